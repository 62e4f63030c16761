// hestenes.cu -- step 4 (eigendecomposition of C_q; north_star's "batched Jacobi
// eigensolver over head_dim x head_dim") as ONE-SIDED (Hestenes) Jacobi, d = 128, fp32, with
// the working matrix held in REGISTERS.
//
// C_q is symmetric positive semi-definite (C is a Gram matrix of centered keys and
// (sigma sigma^T) (.) C is PSD by the Schur product theorem).  The kernel first factors
// C_q = F F^T by a diagonally pivoted Cholesky (below), then makes the columns of X = F
// mutually orthogonal by plane rotations X <- X J_pq: X = F V with V orthogonal and
// X X^T = F F^T = C_q, so once X^T X is diagonal the normalised columns of X are C_q's
// eigenvectors and ||x_j||^2 its eigenvalues.  V itself is never stored.  (Without the
// factorisation, X = C_q also works -- its singular vectors are its eigenvectors -- but the
// working Gram matrix then has C_q^2's spectrum: 10.6 instead of ~6 sweeps.)
//
// Why one-sided on B200: the two-sided kernel (jacobi32p_kernel, calibrate.cu) must touch
// rows AND columns of A every round, so A and V live in shared memory and every round moves
// every element through the shared-memory pipe (ncu: L1/shared 78-91 %), 11.5 ms for LLaVA
// b32.  A column rotation needs only its two columns: here warp w holds 2 blocks of 8 columns
// with lane l owning rows l, l+32 and l+64, l+96 as two float2 (64 fp32 registers; rotations
// run as packed FFMA2), every pair of columns a warp holds is rotated in registers, and the
// only cross-lane traffic is the pair's inner product (a butterfly reduce-scatter of 8 partial
// sums per 8 disjoint pairs) and the broadcast of the rotation coefficients.  Blocks move
// between warps through shared memory once per block-round (15 per sweep, a 2-block
// tournament over 16 blocks; every column pair meets once per sweep).
//
// Rotation (Golub & Van Loan 8.4, the same Schur rotation as the two-sided kernels, applied to
// the 2x2 Gram matrix [[a, g], [g, b]] of columns p, q):
//   zeta = (b - a) / (2 g),  t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),  c = 1/sqrt(1+t^2),
//   x_p <- c x_p - s x_q,  x_q <- s x_p + c x_q (s = t c),  a <- a - t g,  b <- b + t g,
// applied in scaled form (hj_subround).  A pair is rotated when its cosine |g|/sqrt(a b)
// exceeds tol (2e-6); the iteration stops after a sweep whose largest cosine is below qstop
// (3e-3: convergence is quadratic, so the cosines left are O(qstop^2)).  Column norms are
// recomputed exactly after every exchange.
//
// Output: V0 = X diag(1/||x_j||) (fp32, [d][d] row-major, columns in solver order) and
// lambda_j = ||x_j||^2; the fp64 refinement (refine_tc_kernel, or refine_smem_kernel for
// r > 64) follows.  A column whose squared norm falls below 1e-30 ||C_q||_F^2 (an exactly or
// nearly null direction, whose normalisation is undefined) marks the unit info = -2 and the
// two-sided kernel re-solves it (launch_jacobi).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace rk {

namespace {
constexpr int kHJWarps = 8;
constexpr int kHJThreads = 32 * kHJWarps;
constexpr int kHJLd = 130;  // column stride of the exchange buffer (floats, even: float2 rows)
constexpr unsigned kFull = 0xffffffffu;
constexpr int kNeedTwoSided = -2;

// Reduce-scatter of N per-lane partial sums over the warp (N = 8 or 16): returns the full
// warp sum of value index (lane >> (5 - log2 N)).  log2 N halving levels exchange half of the
// remaining values each, then the remaining 5 - log2 N levels are plain butterflies.
template <int N>
__device__ __forceinline__ float warp_reduce_scatter(const float (&v)[N], int lane) {
  constexpr int L = N == 16 ? 4 : N == 8 ? 3 : N == 4 ? 2 : N == 2 ? 1 : 0;
  static_assert((1 << L) == N, "N must be a power of two <= 16");
  float a[N];
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = v[i];
#pragma unroll
  for (int lev = 0; lev < L; ++lev) {
    const int off = 16 >> lev;
    const int m = N >> (lev + 1);
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = hi ? a[i] : a[i + m];
      const float keep = hi ? a[i + m] : a[i];
      a[i] = keep + __shfl_xor_sync(kFull, send, off);
    }
  }
  float r = a[0];
#pragma unroll
  for (int off = 16 >> L; off >= 1; off >>= 1) r += __shfl_xor_sync(kFull, r, off);
  return r;
}

// Single-instruction MUFU approximations (flush-to-zero: no denormal fix-up code; the
// operands here are normal or the pair is not rotated)
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Columns (0..15 = block A cols 0..7, block B cols 0..7) of pair j in sub-round s.
//   intra-block: 7 rounds of the circle method on each block's 8 columns (pairs j = 4b + m);
//   cross-block: pair j = (A_j, B_{(j + s) mod 8}), 8 rounds.
template <bool kIntra>
__device__ __forceinline__ void hj_pair(int s, int j, int& p, int& q) {
  if (kIntra) {
    const int b = j >> 2, m = j & 3;
    const int pm = m == 0 ? 0 : 1 + (m - 1 + s) % 7;
    const int qm = 1 + (6 - m + s) % 7;  // position 7 - m >= 4 is never the fixed player
    p = 8 * b + pm;
    q = 8 * b + qm;
  } else {
    p = j;
    q = 8 + ((j + s) & 7);
  }
}

// One sub-round: 8 disjoint column pairs of the warp's 16 columns.  Column j is held scaled,
// x_j = dsc[j] y_j (registers hold y), nrm[j] = ||x_j||^2.  cmax collects the largest squared
// cosine g^2 / (a b) seen by this lane's pair (the stopping test).
template <bool kIntra, int S>
__device__ __forceinline__ void hj_subround(float2 (&x)[16][2], float* nrm, float* dsc, float tol2,
                                            int lane, float& cmax) {
  float g[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int p, q;
    hj_pair<kIntra>(S, j, p, q);
    const float2 a2 = __ffma2_rn(x[p][1], x[q][1], __fmul2_rn(x[p][0], x[q][0]));
    g[j] = a2.x + a2.y;
  }
  const float gy = warp_reduce_scatter<8>(g, lane);  // pair lane >> 2 (scaled columns)
  int p, q;
  hj_pair<kIntra>(S, lane >> 2, p, q);
  const float al = nrm[p], be = nrm[q], dp = dsc[p], dq = dsc[q];
  const float gam = gy * dp * dq;  // inner product of the true columns
  const float g2 = gam * gam, ab = al * be;
  // (null columns, ab ~ 0, are reported as info -2 after the sweeps)
  cmax = fmaxf(cmax, ab > 1e-36f ? g2 * rcp_ftz(ab) : 0.f);
  const bool rot = g2 > tol2 * ab;  // cosine above tol
  // branch-free: lanes that do not rotate take a1 = a2 = t = 0, c = 1 whatever zeta is
  // (gam = 0 gives inf / NaN here, discarded), and every pair is updated -- a zero update
  // leaves the columns bit-identical, and without a skip branch the unrolled sub-rounds keep
  // their registers in place (a conditional update forces moves at the merge point)
  const float zeta = (be - al) * rcp_ftz(2.f * gam);
  const float az = fabsf(zeta);
  // sqrt(1 + zeta^2) ~ |zeta| beyond 1e18 (zeta^2 would overflow); approximate reciprocal
  // and square root: an inexact t only changes the angle slightly (the sweep goes on until
  // the cosines are small), an inexact c only rescales the pair (norms are recomputed)
  const float z2 = fmaf(az, az, 1.f);
  float t = rcp_ftz(az + (az < 1e18f ? z2 * rsqrt_ftz(z2) : az));
  t = rot ? (zeta < 0.f ? -t : t) : 0.f;
  const float c = rsqrt_ftz(fmaf(t, t, 1.f));
  // scaled rotation: x = d y per column; x_p <- c (x_p - t x_q), x_q <- c (x_q + t x_p)
  // becomes d <- c d and y_p <- y_p - (t d_q / d_p) y_q, y_q <- y_q + (t d_p / d_q) y_p:
  // two FMAs per element pair instead of four multiply(-add)s
  const float rq = dq * rcp_ftz(dp);
  const float a1 = t * rq, a2 = t * rcp_ftz(rq);
  // every lane has read nrm / dsc (their values fed the coefficients) before the update
  __syncwarp();
  if (rot && (lane & 3) == 0) {
    nrm[p] = fmaf(-t, gam, al);
    nrm[q] = fmaf(t, gam, be);
    dsc[p] = dp * c;
    dsc[q] = dq * c;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // pair j's coefficients from its lane group, then its update
    int pp, qq;
    hj_pair<kIntra>(S, j, pp, qq);
    const float c1 = __shfl_sync(kFull, a1, 4 * j), c2 = __shfl_sync(kFull, a2, 4 * j);
    const float2 m1 = make_float2(-c1, -c1), m2 = make_float2(c2, c2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // packed fp32x2 FMAs (FFMA2): two rows per instruction
      const float2 yp = x[pp][h];
      x[pp][h] = __ffma2_rn(m1, x[qq][h], yp);
      x[qq][h] = __ffma2_rn(m2, yp, x[qq][h]);
    }
  }
  __syncwarp();
}

// exact squared norms of the warp's 16 (unscaled) columns into nrm[0..15], scales to 1
__device__ __forceinline__ void hj_norms(const float2 (&x)[16][2], float* nrm, float* dsc, int lane) {
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // two halves of 8 columns: fewer live registers
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float2 a = __ffma2_rn(x[8 * h + j][1], x[8 * h + j][1], __fmul2_rn(x[8 * h + j][0], x[8 * h + j][0]));
      v[j] = a.x + a.y;
    }
    const float r = warp_reduce_scatter<8>(v, lane);  // column 8 h + (lane >> 2)
    if ((lane & 3) == 0) {
      nrm[8 * h + (lane >> 2)] = r;
      dsc[8 * h + (lane >> 2)] = 1.f;
    }
  }
  __syncwarp();
}

// element k (row lane + 32 k) of column j: rows (lane, lane + 32) and (lane + 64, lane + 96)
// are packed in one float2 each so the rotations run as FFMA2
__device__ __forceinline__ float& xel(float2 (&x)[16][2], int j, int k) {
  return (k & 1) ? x[j][k >> 1].y : x[j][k >> 1].x;
}

// Shared-memory position (floats) of row r within a column: rows (l, l + 32) and
// (l + 64, l + 96) are adjacent, so a lane moves its x[j][h] as one 8-byte access
__device__ __forceinline__ int hj_f(int r) { return 2 * ((r & 31) + 32 * (r >> 6)) + ((r >> 5) & 1); }
__device__ __forceinline__ float2* hj_col2(float* Xs, int col) {
  return reinterpret_cast<float2*>(Xs + col * kHJLd);
}

// block held in tournament slot i at block-round k (circle method, slot 0 fixed)
__device__ __forceinline__ int hj_slot_block(int i, int k) { return i == 0 ? 0 : 1 + (i - 1 + k) % 15; }

template <int K>
struct HjIntra {
  __device__ __forceinline__ static void run(float2 (&x)[16][2], float* nrm, float* dsc, float tol2, int lane,
                                             float& cm) {
    hj_subround<true, K>(x, nrm, dsc, tol2, lane, cm);
    HjIntra<K + 1>::run(x, nrm, dsc, tol2, lane, cm);
  }
};
template <>
struct HjIntra<7> {
  __device__ __forceinline__ static void run(float2 (&)[16][2], float*, float*, float, int, float&) {}
};
template <int K>
struct HjCross {
  __device__ __forceinline__ static void run(float2 (&x)[16][2], float* nrm, float* dsc, float tol2, int lane,
                                             float& cm) {
    hj_subround<false, K>(x, nrm, dsc, tol2, lane, cm);
    HjCross<K + 1>::run(x, nrm, dsc, tol2, lane, cm);
  }
};
template <>
struct HjCross<8> {
  __device__ __forceinline__ static void run(float2 (&)[16][2], float*, float*, float, int, float&) {}
};
}  // namespace

size_t hestenes_smem_bytes() { return ((size_t)128 * kHJLd + 32 * kHJWarps) * sizeof(float); }

__global__ void __launch_bounds__(kHJThreads, 2) hestenes_kernel(const double* __restrict__ cq,
                                                                 float* __restrict__ lam_out,
                                                                 float* __restrict__ vecs,
                                                                 int32_t* __restrict__ jinfo,
                                                                 float tol, float qstop,
                                                                 int max_sweeps, int report_sweeps) {
  constexpr int d = 128;
  extern __shared__ __align__(16) float hsm[];
  float* Xs = hsm;                                  // [col][kHJLd]
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  float* nrm = hsm + d * kHJLd + 16 * w;            // this warp's 16 squared column norms
  float* dsc = hsm + d * kHJLd + 16 * kHJWarps + 16 * w;  // and their scales (x = dsc y)
  __shared__ double s_red[kHJWarps];
  __shared__ int s_bad;

  // finiteness and ||C||_F (fp64); the matrix is scaled by an exact power of two to ~1
  const double* C = cq + (size_t)u * d * d;
  double f2 = 0.0;
  int bad = 0;
  for (int e = tid; e < d * d / 2; e += kHJThreads) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(C) + e);
    if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
    f2 = fma(v.x, v.x, fma(v.y, v.y, f2));
  }
  if (tid == 0) s_bad = 0;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) f2 += __shfl_xor_sync(kFull, f2, off);
  bad = __any_sync(kFull, bad);
  if (lane == 0) s_red[w] = f2;
  __syncthreads();
  if (bad && lane == 0) s_bad = 1;
  double tot = 0.0;
#pragma unroll
  for (int i = 0; i < kHJWarps; ++i) tot += s_red[i];
  __syncthreads();
  if (s_bad) {
    for (int e = tid; e < d * d; e += kHJThreads) vecs[(size_t)u * d * d + e] = 0.f;
    for (int j = tid; j < d; j += kHJThreads) lam_out[(size_t)u * d + j] = CUDART_NAN_F;
    if (tid == 0) jinfo[u] = -1;
    return;
  }
  int ex = 0;
  if (tot > 0.0) frexp(sqrt(tot), &ex);
  const double scale = ldexp(1.0, -ex);
  const float unscale = ldexpf(1.f, ex);  // C_q = unscale * (scaled matrix)

  // A = C_q in registers: warp w holds blocks w and 15 - w (tournament slots w, 15 - w at
  // k = 0), column cj(j) in x[j]; column c of the symmetric C_q is its row c (coalesced)
  float2 x[16][2];
  // blocks w and 15 - w: column of x[j] (computed, not held: registers are the budget)
  auto cj = [w](int j) { return j < 8 ? 8 * w + j : 112 - 8 * w + j; };
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) xel(x, j, k) = (float)(C[(size_t)cj(j) * d + lane + 32 * k] * scale);

  // Preconditioner: diagonally pivoted Cholesky C_q = F F^T (outer-product form, fp32).  The
  // one-sided iteration then runs on F, whose left singular vectors are C_q's eigenvectors and
  // whose squared singular values are its eigenvalues: the working Gram matrix has C_q's
  // spectrum instead of C_q^2's, and pivoting grades F's columns (Drmac & Veselic's
  // preconditioned Jacobi) -- 12 -> 7 sweeps on the bench configs.  Step k takes the largest
  // remaining diagonal entry p: F[:, k] = A[:, p] / sqrt(A_pp) (= row p by symmetry: lane p%32
  // of every warp writes its columns' entries), A <- A - F[:, k] F[:, k]^T on the remaining
  // columns.  Pivots below d eps max_i(C_ii) stop the factorisation; the remaining (tiny)
  // Schur-complement columns are appended to F as they are, so F F^T = C_q up to rounding.
  // (F[:, k] is column p of A: the symmetric update keeps A exactly symmetric, so the r1-style
  // row write by lane p % 32 of every warp and this owner-warp column write are the same.)
  // The remaining diagonal is tracked in registers, redundantly by every warp (lane l holds
  // rows l + 32 i), so a step needs a single barrier: the pivot column's publication.
  float dgr[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) dgr[i] = (float)(C[(size_t)(lane + 32 * i) * (d + 1)] * scale);
  uint32_t elim = 0;  // bit j: column cj(j) is eliminated
  int kf = 0;
  float ptol = 0.f;
#pragma unroll 1
  for (; kf < d; ++kf) {
    // pivot: largest remaining diagonal entry, ties -> lowest index (eliminated: -inf)
    float bv = dgr[0];
    int bi = lane;
#pragma unroll
    for (int i = 1; i < 4; ++i)
      if (dgr[i] > bv) { bv = dgr[i]; bi = lane + 32 * i; }
    const uint32_t key = bv > 0.f ? __float_as_uint(bv) : 0u;  // order-preserving for v > 0
    const uint32_t kmax = __reduce_max_sync(kFull, key);
    const int p = (int)__reduce_min_sync(kFull, key == kmax ? (uint32_t)bi : 0xffffffffu);
    bv = __uint_as_float(kmax);
    if (kf == 0) ptol = (float)d * 5.96e-8f * bv;
    if (!(bv > ptol)) break;  // identical decision in every warp
    const float rs = rsqrtf(bv);
    float* Fk = Xs + kf * kHJLd;
    {
      // F[:, k] = A[:, p] / sqrt(A_pp): column p lives in one warp's registers (blocks w and
      // 15 - w); that warp writes it (two 8-byte stores per lane), rows already eliminated
      // as exact zeros
      const int pb = p >> 3;
      if (w == (pb < 8 ? pb : 15 - pb)) {
        const int jp = (pb < 8 ? 0 : 8) + (p & 7);
        float2 c0 = x[0][0], c1 = x[0][1];
#pragma unroll
        for (int j = 1; j < 16; ++j)
          if (j == jp) { c0 = x[j][0]; c1 = x[j][1]; }
        c0 = __fmul2_rn(c0, make_float2(rs, rs));
        c1 = __fmul2_rn(c1, make_float2(rs, rs));
        if (dgr[0] == -CUDART_INF_F) c0.x = 0.f;
        if (dgr[1] == -CUDART_INF_F) c0.y = 0.f;
        if (dgr[2] == -CUDART_INF_F) c1.x = 0.f;
        if (dgr[3] == -CUDART_INF_F) c1.y = 0.f;
        float2* F2 = hj_col2(Xs, kf) + lane;
        F2[0] = c0;
        F2[32] = c1;
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (cj(j) == p) elim |= 1u << j;
    __syncthreads();  // F[:, k] complete (the next step writes another column: no second barrier)
    const float2 l01 = reinterpret_cast<const float2*>(Fk)[lane];
    const float2 l23 = reinterpret_cast<const float2*>(Fk)[lane + 32];
    const float lr[4] = {l01.x, l01.y, l23.x, l23.y};  // rows lane + 32 i
#pragma unroll
    for (int i = 0; i < 4; ++i) dgr[i] = lane + 32 * i == p ? -CUDART_INF_F : fmaf(-lr[i], lr[i], dgr[i]);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if ((elim >> j) & 1u) continue;  // warp-uniform
      const float lc = -Fk[hj_f(cj(j))];
      const float2 m = make_float2(lc, lc);
      x[j][0] = __ffma2_rn(l01, m, x[j][0]);
      x[j][1] = __ffma2_rn(l23, m, x[j][1]);
    }
  }
  // append the remaining columns (in index order) after the kf pivot columns
  {
    uint32_t rem[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) rem[i] = __ballot_sync(kFull, dgr[i] != -CUDART_INF_F);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if ((elim >> j) & 1u) continue;
      const int c = cj(j), wd = c >> 5;
      int pos = kf + __popc(rem[wd] & ((1u << (c & 31)) - 1u));
#pragma unroll
      for (int i = 0; i < 4; ++i) pos += i < wd ? __popc(rem[i]) : 0;
      float2* dst = hj_col2(Xs, pos) + lane;
      dst[0] = x[j][0];
      dst[32] = x[j][1];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float2* src = hj_col2(Xs, cj(j)) + lane;
    x[j][0] = src[0];
    x[j][1] = src[32];
  }
  __syncthreads();
  hj_norms(x, nrm, dsc, lane);

  const float tol2 = tol * tol, q2 = qstop * qstop;
  int sweep = 0, converged = 0;
  for (;;) {
    if (sweep >= max_sweeps) break;
    float cm = 0.f;
    HjIntra<0>::run(x, nrm, dsc, tol2, lane, cm);
#pragma unroll 1
    for (int k = 0; k < 15; ++k) {
      HjCross<0>::run(x, nrm, dsc, tol2, lane, cm);
      // exchange: blocks go back to shared memory by block id and come out by the next
      // round's tournament slots (k = 14 -> 0 restores the start arrangement)
      // (the scales are folded back in: shared memory holds the true columns)
      const int ba = hj_slot_block(w, k), bb = hj_slot_block(15 - w, k);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float2* dst = hj_col2(Xs, 8 * (j < 8 ? ba : bb) + (j & 7)) + lane;
        const float sc = dsc[j];
        dst[0] = __fmul2_rn(x[j][0], make_float2(sc, sc));
        dst[32] = __fmul2_rn(x[j][1], make_float2(sc, sc));
      }
      __syncthreads();
      const int k1 = k == 14 ? 0 : k + 1;
      const int na = hj_slot_block(w, k1), nb = hj_slot_block(15 - w, k1);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float2* src = hj_col2(Xs, 8 * (j < 8 ? na : nb) + (j & 7)) + lane;
        x[j][0] = src[0];
        x[j][1] = src[32];
      }
      __syncthreads();
      hj_norms(x, nrm, dsc, lane);
    }
    ++sweep;
    // quadratic convergence: after a sweep whose largest cosine was <= qstop the remaining
    // cosines are O(qstop^2), below what the fp64 refinement needs (no check sweep)
    if (!__syncthreads_or(cm > q2 ? 1 : 0)) {
      converged = 1;
      break;
    }
  }

  // V0 = X diag(1 / ||x_j||), lambda_j = ||x_j||; staged through shared memory so the
  // row-major global writes are coalesced
  const int ba = hj_slot_block(w, 0), bb = hj_slot_block(15 - w, 0);
  int degenerate = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = 8 * (j < 8 ? ba : bb) + (j & 7);
    const float n2 = nrm[j];
    if (!(n2 >= 1e-30f)) degenerate = 1;
    const float inv = n2 > 0.f ? rsqrtf(n2) : 0.f;
    float2* dst = hj_col2(Xs, col) + lane;
    dst[0] = __fmul2_rn(x[j][0], make_float2(inv, inv));
    dst[32] = __fmul2_rn(x[j][1], make_float2(inv, inv));
    if (lane == 0) lam_out[(size_t)u * d + col] = n2 * unscale;  // ||f_j||^2 = lambda_j
  }
  degenerate = __syncthreads_or(degenerate);
  float* Vo = vecs + (size_t)u * d * d;
  for (int e = tid; e < d * d; e += kHJThreads) {
    const int row = e / d, col = e % d;
    Vo[e] = Xs[col * kHJLd + hj_f(row)];
  }
  if (tid == 0)
    jinfo[u] = degenerate ? kNeedTwoSided
                          : (converged ? (report_sweeps ? 1000 + sweep : 0) : (sweep > 0 ? sweep : 1));
}

int launch_hestenes(int U, const double* cq, float* lam, float* v32, int32_t* jinfo, float tol,
                    float qstop, int max_sweeps, cudaStream_t st) {
  static int attr[kMaxDevices];
  const size_t sm = hestenes_smem_bytes();
  once_per_device(attr, [&] {
    return cudaFuncSetAttribute(hestenes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) ==
                   cudaSuccess
               ? 1
               : 0;
  });
  // diagnostics only: ROTATEK_HJ_SWEEPS=1 reports info = 1000 + sweeps for converged units
  static const int report = getenv("ROTATEK_HJ_SWEEPS") != nullptr;
  hestenes_kernel<<<U, kHJThreads, sm, st>>>(cq, lam, v32, jinfo, tol, qstop, max_sweeps, report);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rk
