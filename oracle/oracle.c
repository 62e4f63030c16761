/*
 * oracle.c -- plain, slow, fp64 CPU oracle for the RotateK hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path under
 * paper_2605_19218_b200/, and it never reads anything the CUDA path produced
 * except where a test explicitly hands it "the bytes the GPU holds" as inputs.
 *
 * Citations "P:<line>" are lines of the paper's LaTeX source:
 *   Alg. 1 = alg:rotatek-prefill
 *   Alg. 2 = alg:rotatek-decode
 *   Sec. 3.2 query-weighted PCA
 *   Sec. 3.3 post-hoc reweighting
 *   App. C decode kernel
 * Readings of silent / ambiguous passages are listed in DESIGN.md ("Readings").
 *
 * Everything is double precision, plain loops, no blocking, no reordering
 * beyond what the stated definition needs.  OpenMP parallelises only over
 * independent units (batch x kv-head), never inside one unit's arithmetic.
 *
 * Pins: every function here is checked by tests/test_oracle_*.py against
 * hand values (tests/golden/), closed forms, numpy.linalg.eigh (library
 * special case), brute force on tiny inputs and exact invariants.  No
 * function is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IDX2(i, j, ld) ((size_t)(i) * (size_t)(ld) + (size_t)(j))

int orc_abi_version(void) { return 1; }

/* ------------------------------------------------------------------------ */
/* Step 1: query-window norms.  (sigma_W)_j = ||(Q_W)_{:,j}||_2  (*/
/* Alg. 1 line "sigma_j <- ||(Q_W)_{:,j}||_2").  Reading Q4: under   */
/* GQA the window of a KV unit is the concatenation of its G query heads'   */
/* W rows, so the norm runs over G*W rows.  W == 0 -> sigma == 1 (query-    */
/* agnostic mode, the K-only PCA arm of tab:rotatek-ablation P:638-641).    */
/* Qw layout [U][G][W][d].                                                  */
/* ------------------------------------------------------------------------ */
void orc_query_sigma(const double* Qw, int U, int G, int W, int d, double* sigma) {
#pragma omp parallel for schedule(static)
  for (int u = 0; u < U; ++u) {
    for (int j = 0; j < d; ++j) {
      if (W == 0) { sigma[IDX2(u, j, d)] = 1.0; continue; }
      double ss = 0.0;
      for (int g = 0; g < G; ++g)
        for (int w = 0; w < W; ++w) {
          double x = Qw[(((size_t)u * G + g) * W + w) * d + j];
          ss += x * x;
        }
      sigma[IDX2(u, j, d)] = sqrt(ss);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Step 2: per-channel mean and centered covariance, two-pass.              */
/*   mu = (1/N) sum_n K_n ;  Kbar = K - 1 mu^T ;  C = Kbar^T Kbar            */
/* (Alg. 1 lines 1-3; Sec. 3.2 "C = (K - mu)^T (K - mu)").*/
/* center == 0 gives mu = 0 and C = K^T K (the north_star's literal         */
/* "Key covariance K^T K"; reading N1 in DESIGN.md).  No 1/N scaling        */
/* (reading Q3).  K layout [U][N][d]; mu [U][d]; C [U][d][d].               */
/* ------------------------------------------------------------------------ */
void orc_mean_cov(const double* K, int U, int N, int d, int center, double* mu, double* C) {
#pragma omp parallel for schedule(static)
  for (int u = 0; u < U; ++u) {
    const double* Ku = K + (size_t)u * N * d;
    double* mu_u = mu + (size_t)u * d;
    double* Cu = C + (size_t)u * d * d;
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      if (center) {
        for (int n = 0; n < N; ++n) s += Ku[IDX2(n, j, d)];
        s /= (double)N;
      }
      mu_u[j] = s;
    }
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        double s = 0.0;
        for (int n = 0; n < N; ++n)
          s += (Ku[IDX2(n, i, d)] - mu_u[i]) * (Ku[IDX2(n, j, d)] - mu_u[j]);
        Cu[IDX2(i, j, d)] = s;
      }
  }
}

/* ------------------------------------------------------------------------ */
/* Step 3: post-hoc reweighting, C_q = (sigma sigma^T) (.) C                */
/* (Sec. 3.3 Hadamard identity; Alg. 1 line 5), followed  */
/* by symmetrisation (C + C^T)/2.  In place on C.                           */
/* ------------------------------------------------------------------------ */
void orc_hadamard(double* C, const double* sigma, int U, int d) {
#pragma omp parallel for schedule(static)
  for (int u = 0; u < U; ++u) {
    double* Cu = C + (size_t)u * d * d;
    const double* s = sigma + (size_t)u * d;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) Cu[IDX2(i, j, d)] *= s[i] * s[j];
    for (int i = 0; i < d; ++i)
      for (int j = i + 1; j < d; ++j) {
        double a = 0.5 * (Cu[IDX2(i, j, d)] + Cu[IDX2(j, i, d)]);
        Cu[IDX2(i, j, d)] = a;
        Cu[IDX2(j, i, d)] = a;
      }
  }
}

/* ------------------------------------------------------------------------ */
/* Step 4: eigendecomposition C_q = R Lambda R^T  ("columns of R are */
/* eigenvectors of C_q").  Textbook cyclic-by-row Jacobi: for every pair     */
/* p<q compute the symmetric Schur rotation that annihilates a_pq and apply */
/* A <- J^T A J, V <- V J; sweep until off(A) <= tol * ||A||_F.             */
/* Solver order: eigenvalue i is the final diagonal entry i, eigenvector i  */
/* is column i of V.  Sign convention: the largest-|entry| of each column is*/
/* made positive (it affects no output).  Returns the number of sweeps, or  */
/* -(sweeps) if not converged within max_sweeps, or -1000000 on non-finite */
/* input.  A is d x d (read only), lam [d], V [d][d].                       */
/* ------------------------------------------------------------------------ */
int orc_jacobi(const double* A_in, int d, double tol, int max_sweeps, double* lam, double* V) {
  double* A = (double*)malloc(sizeof(double) * (size_t)d * d);
  double fro = 0.0;
  for (size_t i = 0; i < (size_t)d * d; ++i) {
    A[i] = A_in[i];
    if (!isfinite(A[i])) { free(A); return -1000000; }
    fro += A[i] * A[i];
  }
  fro = sqrt(fro);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) V[IDX2(i, j, d)] = (i == j) ? 1.0 : 0.0;

  int sweeps = 0, converged = 0;
  for (;;) {
    double off = 0.0;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j)
        if (i != j) off += A[IDX2(i, j, d)] * A[IDX2(i, j, d)];
    off = sqrt(off);
    if (off <= tol * fro) { converged = 1; break; }
    if (sweeps >= max_sweeps) break;
    for (int p = 0; p < d - 1; ++p)
      for (int q = p + 1; q < d; ++q) {
        double apq = A[IDX2(p, q, d)];
        if (apq == 0.0) continue;
        /* symmetric Schur 2x2: tau = (a_qq - a_pp) / (2 a_pq),
           t = sign(tau) / (|tau| + sqrt(1 + tau^2)), c = 1/sqrt(1+t^2), s = t c */
        double tau = (A[IDX2(q, q, d)] - A[IDX2(p, p, d)]) / (2.0 * apq);
        double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = t * c;
        /* A <- J^T A : rows p, q */
        for (int k = 0; k < d; ++k) {
          double ap = A[IDX2(p, k, d)], aq = A[IDX2(q, k, d)];
          A[IDX2(p, k, d)] = c * ap - s * aq;
          A[IDX2(q, k, d)] = s * ap + c * aq;
        }
        /* A <- A J : columns p, q */
        for (int k = 0; k < d; ++k) {
          double ap = A[IDX2(k, p, d)], aq = A[IDX2(k, q, d)];
          A[IDX2(k, p, d)] = c * ap - s * aq;
          A[IDX2(k, q, d)] = s * ap + c * aq;
        }
        /* V <- V J */
        for (int k = 0; k < d; ++k) {
          double vp = V[IDX2(k, p, d)], vq = V[IDX2(k, q, d)];
          V[IDX2(k, p, d)] = c * vp - s * vq;
          V[IDX2(k, q, d)] = s * vp + c * vq;
        }
      }
    ++sweeps;
  }
  for (int i = 0; i < d; ++i) lam[i] = A[IDX2(i, i, d)];
  for (int j = 0; j < d; ++j) {
    int arg = 0;
    double best = -1.0;
    for (int i = 0; i < d; ++i)
      if (fabs(V[IDX2(i, j, d)]) > best) { best = fabs(V[IDX2(i, j, d)]); arg = i; }
    if (V[IDX2(arg, j, d)] < 0.0)
      for (int i = 0; i < d; ++i) V[IDX2(i, j, d)] = -V[IDX2(i, j, d)];
  }
  free(A);
  return converged ? sweeps : -(sweeps > 0 ? sweeps : 1);
}

/* ------------------------------------------------------------------------ */
/* Step 5: top-r select.  "ordered by decreasing eigenvalue magnitude. The  */
/* first k columns are retained".  Reading Q7: order by signed value*/
/* (C_q is PSD).  Reading Q8: ties -> lower solver index; kept columns are  */
/* listed in ascending index.  keep = the first r indices of the order      */
/* (lambda descending, index ascending).  mask bit i <=> i kept; mask has   */
/* ceil(d/32) words, bit i%32 of word i/32.  Returns 0, or -1 on NaN.       */
/* ------------------------------------------------------------------------ */
int orc_select_topr(const double* lam, int d, int r, uint32_t* mask, int32_t* idx) {
  for (int i = 0; i < d; ++i)
    if (isnan(lam[i])) return -1;
  int* order = (int*)malloc(sizeof(int) * (size_t)d);
  for (int i = 0; i < d; ++i) order[i] = i;
  /* insertion sort by (lambda desc, index asc): stable and obviously correct */
  for (int i = 1; i < d; ++i) {
    int x = order[i], j = i - 1;
    while (j >= 0 && lam[order[j]] < lam[x]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = x;
  }
  int words = (d + 31) / 32;
  for (int w = 0; w < words; ++w) mask[w] = 0u;
  for (int k = 0; k < r; ++k) mask[order[k] / 32] |= 1u << (order[k] % 32);
  int n = 0;
  for (int i = 0; i < d; ++i)
    if (mask[i / 32] & (1u << (i % 32))) idx[n++] = i;
  free(order);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Step 6: R_k = R[:, idx] ("R_k collects the top-k columns of R")   */
/* and the mean residual delta_mu = mu - R_k R_k^T mu  (Alg. 1;      */
/* Sec. 3.2 bias "(I_d - R_k R_k^T) mu").  V [d][d], Rr [d][r].      */
/* ------------------------------------------------------------------------ */
void orc_rotation(const double* V, const int32_t* idx, int d, int r, const double* mu,
                  double* Rr, double* dmu) {
  for (int i = 0; i < d; ++i)
    for (int k = 0; k < r; ++k) Rr[IDX2(i, k, r)] = V[IDX2(i, idx[k], d)];
  double* proj = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int k = 0; k < r; ++k) {
    double s = 0.0;
    for (int i = 0; i < d; ++i) s += Rr[IDX2(i, k, r)] * mu[i];
    proj[k] = s;
  }
  for (int i = 0; i < d; ++i) {
    double s = 0.0;
    for (int k = 0; k < r; ++k) s += Rr[IDX2(i, k, r)] * proj[k];
    dmu[i] = mu[i] - s;
  }
  free(proj);
}

/* delta_mu from a given R_r (used for the "as stored" mode, where R_r is   */
/* the rotation the GPU holds): same formula as above.                      */
void orc_dmu_from_R(const double* Rr, int U, int d, int r, const double* mu, double* dmu) {
#pragma omp parallel for schedule(static)
  for (int u = 0; u < U; ++u) {
    const double* R = Rr + (size_t)u * d * r;
    const double* m = mu + (size_t)u * d;
    double* out = dmu + (size_t)u * d;
    for (int i = 0; i < d; ++i) {
      double s = 0.0;
      for (int k = 0; k < r; ++k) {
        double pk = 0.0;
        for (int j = 0; j < d; ++j) pk += R[IDX2(j, k, r)] * m[j];
        s += R[IDX2(i, k, r)] * pk;
      }
      out[i] = m[i] - s;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Full Alg. 1 steps 1-6 over U units (exact eigendecomposition arm,        */
/* "eigh, Q-aware" of tab:rotatek-ablation; reading N2/Q1).          */
/* Outputs: sigma[U][d], mu[U][d], Cq[U][d][d], lam[U][d] (solver order),   */
/* Vfull[U][d][d], mask[U][ceil(d/32)], idx[U][r], Rr[U][d][r], dmu[U][d],  */
/* sweeps[U] (orc_jacobi return code).  Returns 0, or -1 if any unit hit a  */
/* NaN in select.                                                            */
/* ------------------------------------------------------------------------ */
int orc_calibrate(const double* K, const double* Qw, int U, int G, int N, int d, int W, int r,
                  int center, int query_weight, double tol, int max_sweeps,
                  double* sigma, double* mu, double* Cq, double* lam, double* Vfull,
                  uint32_t* mask, int32_t* idx, double* Rr, double* dmu, int32_t* sweeps) {
  orc_query_sigma(Qw, U, G, query_weight ? W : 0, d, sigma);
  orc_mean_cov(K, U, N, d, center, mu, Cq);
  orc_hadamard(Cq, sigma, U, d);
  int words = (d + 31) / 32;
  int bad = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
  for (int u = 0; u < U; ++u) {
    double* Vu = Vfull + (size_t)u * d * d;
    double* lu = lam + (size_t)u * d;
    sweeps[u] = orc_jacobi(Cq + (size_t)u * d * d, d, tol, max_sweeps, lu, Vu);
    if (orc_select_topr(lu, d, r, mask + (size_t)u * words, idx + (size_t)u * r) != 0) {
      bad = 1;
      continue;
    }
    orc_rotation(Vu, idx + (size_t)u * r, d, r, mu + (size_t)u * d, Rr + (size_t)u * d * r,
                 dmu + (size_t)u * d);
  }
  return bad ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* Step 7: K~ = K R_k ("stored in place of K", Alg. 1 line 14), in   */
/* fp64 over uncentered K (reading Q10).  The quantisation point (rounding  */
/* to the cache dtype) is a separate function below.  K [U][N][d],          */
/* Rr [U][d][r], Kt [U][N][r].                                              */
/* ------------------------------------------------------------------------ */
void orc_compress(const double* K, const double* Rr, int U, int N, int d, int r, double* Kt) {
#pragma omp parallel for schedule(static)
  for (int u = 0; u < U; ++u) {
    const double* Ku = K + (size_t)u * N * d;
    const double* R = Rr + (size_t)u * d * r;
    double* out = Kt + (size_t)u * N * r;
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < r; ++k) {
        double s = 0.0;
        for (int i = 0; i < d; ++i) s += Ku[IDX2(n, i, d)] * R[IDX2(i, k, r)];
        out[IDX2(n, k, r)] = s;
      }
  }
}

/* Round-to-nearest-even of a double to the nearest bfloat16 value          */
/* (1 sign, 8 exponent, 7 fraction bits: precision p = 8, e_min = -126,     */
/* subnormal quantum 2^-133, max finite (2 - 2^-7) 2^127).  Written from the */
/* definition: q = 2^(max(e, -126) - 7) with |x| in [2^e, 2^(e+1)), then     */
/* x -> nearbyint(x / q) * q (ties to even under the default rounding mode); */
/* results beyond the largest finite value become +-inf.                    */
double orc_round_bf16(double x) {
  if (!isfinite(x) || x == 0.0) return x;
  int e;
  frexp(fabs(x), &e);   /* |x| = f * 2^e, f in [0.5, 1) -> |x| in [2^(e-1), 2^e) */
  int ex = e - 1;       /* |x| in [2^ex, 2^(ex+1)) */
  if (ex < -126) ex = -126;
  double q = ldexp(1.0, ex - 7);
  double y = nearbyint(x / q) * q;
  double maxf = ldexp(2.0 - ldexp(1.0, -7), 127);
  if (fabs(y) > maxf) return x > 0 ? INFINITY : -INFINITY;
  return y;
}

void orc_round_bf16_array(const double* x, size_t n, double* y) {
  for (size_t i = 0; i < n; ++i) y[i] = orc_round_bf16(x[i]);
}

/* Round-to-nearest-even to IEEE binary32 (C's conversion under the default */
/* rounding mode).                                                           */
void orc_round_f32_array(const double* x, size_t n, double* y) {
  for (size_t i = 0; i < n; ++i) y[i] = (double)(float)x[i];
}

/* ------------------------------------------------------------------------ */
/* Step 8: Alg. 2 decode for every unit u and query head g:     */
/*   q~ = q R_k ; b = q^T delta_mu                                           */
/*   s_vis = (q~ K~^T + b 1^T) * scale ; s_pt = q K_pt^T * scale             */
/*   s = [s_vis ; s_pt] ; out = softmax(s) [V_vis ; V_pt]                    */
/* scale = 1/sqrt(d) when scale <= 0 (Alg. 2 line 3 divides by sqrt(d), not */
/* sqrt(k); reading Q12).  The softmax subtracts max(s) (a shift that leaves */
/* it unchanged) and divides by the plain sum (epsilon = 0, reading Q13).    */
/* q [U][G][d], Kt [U][N][r], V [U][N][d], Rr [U][d][r], dmu [U][d] (may be  */
/* NULL = zero), Ktext/Vtext [U][M][d], out [U][G][d].  Query head h = u*G+g */
/* maps to KV head u (h_kv = floor(h/G), App. C).                     */
/* ------------------------------------------------------------------------ */
static void scores_one(int u, int g, int G, int d, int r, int N, int M, const double* q,
                       const double* Kt, const double* Rr, const double* dmu,
                       const double* Ktext, double scale, double* s) {
  const double* qv = q + ((size_t)u * G + g) * d;
  const double* R = Rr + (size_t)u * d * r;
  double* qt = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int k = 0; k < r; ++k) { /* Alg. 2 line 1: q~ = q R_k */
    double a = 0.0;
    for (int i = 0; i < d; ++i) a += qv[i] * R[IDX2(i, k, r)];
    qt[k] = a;
  }
  double b = 0.0; /* Alg. 2 line 2: b = q^T delta_mu */
  if (dmu)
    for (int i = 0; i < d; ++i) b += qv[i] * dmu[(size_t)u * d + i];
  for (int n = 0; n < N; ++n) { /* line 3: s_vis = (q~ K~^T + b) / sqrt(d) */
    double a = 0.0;
    for (int k = 0; k < r; ++k) a += qt[k] * Kt[((size_t)u * N + n) * r + k];
    s[n] = (a + b) * scale;
  }
  for (int m = 0; m < M; ++m) { /* line 4: s_pt = q K_pt^T / sqrt(d) */
    double a = 0.0;
    for (int i = 0; i < d; ++i) a += qv[i] * Ktext[((size_t)u * M + m) * d + i];
    s[N + m] = a * scale;
  }
  free(qt);
}

/* Scores only (lines 1-5 of Alg. 2): s [U][G][N+M]. */
void orc_scores(int U, int G, int d, int r, int N, int M, const double* q, const double* Kt,
                const double* Rr, const double* dmu, const double* Ktext, double scale,
                double* s) {
  if (scale <= 0.0) scale = 1.0 / sqrt((double)d);
#pragma omp parallel for collapse(2) schedule(static)
  for (int u = 0; u < U; ++u)
    for (int g = 0; g < G; ++g)
      scores_one(u, g, G, d, r, N, M, q, Kt, Rr, dmu, Ktext, scale,
                 s + ((size_t)u * G + g) * (size_t)(N + M));
}

void orc_decode(int U, int G, int d, int r, int N, int M, const double* q, const double* Kt,
                const double* V, const double* Rr, const double* dmu, const double* Ktext,
                const double* Vtext, double scale, double* out) {
  if (scale <= 0.0) scale = 1.0 / sqrt((double)d);
#pragma omp parallel for collapse(2) schedule(static)
  for (int u = 0; u < U; ++u)
    for (int g = 0; g < G; ++g) {
      double* o = out + ((size_t)u * G + g) * d;
      double* s = (double*)malloc(sizeof(double) * (size_t)(N + M > 0 ? N + M : 1));
      scores_one(u, g, G, d, r, N, M, q, Kt, Rr, dmu, Ktext, scale, s);
      /* lines 5-6: softmax over the concatenation, weighted sum of values */
      double mx = -INFINITY;
      for (int t = 0; t < N + M; ++t)
        if (s[t] > mx) mx = s[t];
      double den = 0.0;
      for (int t = 0; t < N + M; ++t) {
        s[t] = exp(s[t] - mx);
        den += s[t];
      }
      for (int i = 0; i < d; ++i) {
        double a = 0.0;
        for (int n = 0; n < N; ++n) a += s[n] * V[((size_t)u * N + n) * d + i];
        for (int m = 0; m < M; ++m) a += s[N + m] * Vtext[((size_t)u * M + m) * d + i];
        o[i] = a / den;
      }
      free(s);
    }
}

/* ------------------------------------------------------------------------ */
/* NEXT-1: the paper's default solver, Cholesky-QR subspace iteration        */
/* (Alg. 1 lines 6-13; Sec. 3.3; App. E):               */
/*   V <- V0 (given: "Sample V with i.i.d. N(0,1) entries" -- the random     */
/*        numbers are an input so both sides use the same draw)               */
/*   repeat T times:  V <- C_q V ; G <- V^T V ; rho <- eps tr(G) / k ;         */
/*                    L <- Cholesky(G + rho I) ; V <- V L^{-T}                 */
/*   R_k <- V                                                                 */
/* One unit: C [d][d], V0 [d][k], out Rk [d][k].  Returns 0, or -1 if a       */
/* Cholesky pivot is not positive.                                           */
/* ------------------------------------------------------------------------ */
int orc_subspace(const double* C, const double* V0, int d, int k, int T, double eps, double* Rk) {
  double* V = (double*)malloc(sizeof(double) * (size_t)d * k);
  double* W = (double*)malloc(sizeof(double) * (size_t)d * k);
  double* G = (double*)malloc(sizeof(double) * (size_t)k * k);
  double* L = (double*)calloc((size_t)k * k, sizeof(double));
  int rc = 0;
  memcpy(V, V0, sizeof(double) * (size_t)d * k);
  for (int t = 0; t < T && rc == 0; ++t) {
    for (int i = 0; i < d; ++i) /* V <- C V */
      for (int j = 0; j < k; ++j) {
        double s = 0.0;
        for (int l = 0; l < d; ++l) s += C[IDX2(i, l, d)] * V[IDX2(l, j, k)];
        W[IDX2(i, j, k)] = s;
      }
    for (int a = 0; a < k; ++a) /* G <- V^T V */
      for (int b = 0; b < k; ++b) {
        double s = 0.0;
        for (int i = 0; i < d; ++i) s += W[IDX2(i, a, k)] * W[IDX2(i, b, k)];
        G[IDX2(a, b, k)] = s;
      }
    double tr = 0.0; /* rho <- eps tr(G) / k */
    for (int a = 0; a < k; ++a) tr += G[IDX2(a, a, k)];
    const double rho = eps * tr / (double)k;
    for (int a = 0; a < k; ++a) G[IDX2(a, a, k)] += rho;
    for (int j = 0; j < k && rc == 0; ++j) { /* L <- Cholesky(G + rho I), G = L L^T */
      double s = G[IDX2(j, j, k)];
      for (int m = 0; m < j; ++m) s -= L[IDX2(j, m, k)] * L[IDX2(j, m, k)];
      if (!(s > 0.0)) { rc = -1; break; }
      L[IDX2(j, j, k)] = sqrt(s);
      for (int i = j + 1; i < k; ++i) {
        double v = G[IDX2(i, j, k)];
        for (int m = 0; m < j; ++m) v -= L[IDX2(i, m, k)] * L[IDX2(j, m, k)];
        L[IDX2(i, j, k)] = v / L[IDX2(j, j, k)];
      }
    }
    if (rc) break;
    for (int i = 0; i < d; ++i) /* V <- W L^{-T}: each row x solves x L^T = w */
      for (int j = 0; j < k; ++j) {
        double s = W[IDX2(i, j, k)];
        for (int m = 0; m < j; ++m) s -= V[IDX2(i, m, k)] * L[IDX2(j, m, k)];
        V[IDX2(i, j, k)] = s / L[IDX2(j, j, k)];
      }
  }
  memcpy(Rk, V, sizeof(double) * (size_t)d * k);
  free(V); free(W); free(G); free(L);
  return rc;
}

/* KV-budget multiplier of tab:main_comparison: keys pruned to  */
/* channel_keep of their channels, values kept full, so the visual cache    */
/* shrinks by token_keep * (1 + channel_keep) / 2.                           */
double orc_budget(double token_keep, double channel_keep) {
  return token_keep * (1.0 + channel_keep) / 2.0;
}
