// subspace.cu -- NEXT-1: the paper's default solver, Cholesky-QR subspace iteration
// (Alg. 1 lines 6-13; Sec. 3.3):
//   V <- V0;  T times: V <- C_q V; G <- V^T V; rho <- eps tr(G)/k; L <- chol(G + rho I);
//   V <- V L^{-T};  R_k <- V;  delta_mu <- mu - R_k R_k^T mu (computed from the stored R_k)
// The paper issues four kernels per iteration (two GEMMs, Cholesky, triangular solve) and
// captures the T-step loop in a CUDA graph; here the whole loop for every (batch, KV head)
// unit is ONE kernel: one CTA per unit keeps V, C_q V, G and L in shared memory (fp64), so
// the solve costs one launch regardless of T.
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace rk {

namespace {
constexpr int kSubThreads = 256;
}

size_t subspace_smem_bytes(int d, int k) {
  const int ldv = k + 1;  // padded row stride (conflict-free per-row access in the solve)
  return ((size_t)2 * d * ldv + 2 * (size_t)k * k + 64) * sizeof(double);
}

template <int K>
__global__ void __launch_bounds__(kSubThreads) subspace_kernel(int d, int iters, double eps,
                                                               const double* __restrict__ cq,
                                                               const double* __restrict__ mu,
                                                               const float* __restrict__ V0,
                                                               bool center, float* __restrict__ R,
                                                               float* __restrict__ dmu,
                                                               float* __restrict__ ritz,
                                                               int32_t* __restrict__ info) {
  extern __shared__ __align__(16) double ssm[];
  constexpr int ldv = K + 1;
  double* V = ssm;               // [d][ldv]
  double* W = V + d * ldv;       // [d][ldv]   C V
  double* G = W + d * ldv;       // [K][K]
  double* L = G + K * K;         // [K][K]     lower Cholesky factor
  double* red = L + K * K;       // [64]
  __shared__ int s_bad;
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* C = cq + (size_t)u * d * d;
  if (tid == 0) s_bad = 0;
  for (int e = tid; e < d * K; e += blockDim.x) V[(e / K) * ldv + e % K] = (double)V0[(size_t)u * d * K + e];
  __syncthreads();

  auto mul_CV = [&]() {  // W = C V  (4 x 4 output tiles, C from L2)
    constexpr int KT = K / 4;
    for (int t = tid; t < (d / 4) * KT; t += blockDim.x) {
      const int i0 = (t / KT) * 4, j0 = (t % KT) * 4;
      double acc[4][4] = {};
      for (int l = 0; l < d; ++l) {
        double cv[4], vv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) cv[a] = __ldg(C + (size_t)(i0 + a) * d + l);
#pragma unroll
        for (int b = 0; b < 4; ++b) vv[b] = V[l * ldv + j0 + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(cv[a], vv[b], acc[a][b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) W[(i0 + a) * ldv + j0 + b] = acc[a][b];
    }
  };

  for (int it = 0; it < iters; ++it) {
    mul_CV();
    __syncthreads();
    // G = W^T W
    for (int e = tid; e < K * K; e += blockDim.x) {
      const int a = e / K, b = e % K;
      double s = 0.0;
      if (a <= b) {
        for (int i = 0; i < d; ++i) s = fma(W[i * ldv + a], W[i * ldv + b], s);
        G[a * K + b] = s;
        G[b * K + a] = s;
      }
    }
    __syncthreads();
    // rho = eps tr(G) / k ; L = chol(G + rho I)  (warp 0, lanes over rows)
    if (warp == 0) {
      double tr = 0.0;
      for (int a = lane; a < K; a += 32) tr += G[a * K + a];
      tr = warp_sum(tr);
      const double rho = eps * tr / (double)K;
      for (int j = 0; j < K; ++j) {
        double s = G[j * K + j] + rho;
        for (int m = 0; m < j; ++m) s -= L[j * K + m] * L[j * K + m];
        if (!(s > 0.0)) {
          if (lane == 0) s_bad = 1;
          s = 1.0;
        }
        const double ljj = sqrt(s);
        for (int i = j + 1 + lane; i < K; i += 32) {
          double v = G[i * K + j];
          for (int m = 0; m < j; ++m) v -= L[i * K + m] * L[j * K + m];
          L[i * K + j] = v / ljj;
        }
        if (lane == 0) L[j * K + j] = ljj;
        __syncwarp();
      }
    }
    __syncthreads();
    // V = W L^{-T}: every row x solves x L^T = w (forward substitution)
    for (int i = tid; i < d; i += blockDim.x) {
      for (int j = 0; j < K; ++j) {
        double s = W[i * ldv + j];
        for (int m = 0; m < j; ++m) s -= V[i * ldv + m] * L[j * K + m];
        V[i * ldv + j] = s / L[j * K + j];
      }
    }
    __syncthreads();
  }
  // store R = V rounded to fp32; delta_mu from the stored values (fp64)
  float* Ru = R + (size_t)u * d * K;
  for (int e = tid; e < d * K; e += blockDim.x) {
    const float v = (float)V[(e / K) * ldv + e % K];
    Ru[e] = v;
    V[(e / K) * ldv + e % K] = (double)v;
  }
  __syncthreads();
  if (tid < K) {
    double s = 0.0;
    if (center)
      for (int x = 0; x < d; ++x) s = fma(V[x * ldv + tid], mu[(size_t)u * d + x], s);
    red[tid] = s;
  }
  __syncthreads();
  for (int x = tid; x < d; x += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = fma(V[x * ldv + k], red[k], s);
    dmu[(size_t)u * d + x] = center ? (float)(mu[(size_t)u * d + x] - s) : 0.f;
  }
  // Rayleigh quotients of the returned basis: ritz_j = R_j^T C R_j / R_j^T R_j
  if (ritz) {
    __syncthreads();
    mul_CV();
    __syncthreads();
    for (int j = tid; j < K; j += blockDim.x) {
      double num = 0.0, den = 0.0;
      for (int i = 0; i < d; ++i) {
        num = fma(V[i * ldv + j], W[i * ldv + j], num);
        den = fma(V[i * ldv + j], V[i * ldv + j], den);
      }
      ritz[(size_t)u * K + j] = (float)(num / den);
    }
  }
  if (tid == 0 && info) info[u] = s_bad ? -1 : 0;
}

// ------------------------------------------------------------------------------------------
// d = 128: the two GEMMs of every iteration (W = C_q V and G = W^T W) and the final Rayleigh
// quotients on the fp64 tensor cores (DMMA, mma.sync.m8n8k4.f64: fp64 products and sums, so
// the iteration stays an fp64 one, as the oracle's).  Warp w owns rows [16w, 16w + 16) of
// W = C_q V and reads its 16 rows of C_q straight from global memory once per iteration
// (L2-resident after the first: the SM's units hold ~0.25 MB); V, W, G, L stay in shared
// memory with row strides = 4 (mod 16) doubles, which makes every DMMA operand load of a
// half-warp hit 32 distinct banks.  Two CTAs per SM: one's serial phases (Cholesky,
// substitution) overlap the other's GEMMs.
namespace {
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
constexpr int kTcD = 128;
// 1/sqrt(x) for a positive normal x: the hardware approximation (rel. error < 2^-22.9) and two
// Newton steps (fp64-accurate) -- no slow-path call, so no register spills in the Cholesky
__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  y = y * fma(-0.5 * x, y * y, 1.5);
  return y;
}
// Cholesky of a KB x KB (KB <= 32) symmetric block (rows `src`, stride ld; lower triangle read)
// by one warp, lane i holding row i in registers, right-looking: at step j lane j's diagonal
// gives l_jj, the lanes below scale their l_ij and publish the column, and every row
// subtracts l_ij l_kj from its entries k > j (column j read back as shared-memory broadcasts;
// rows above k only touch their unused upper part).  Writes L (zero upper part) and 1/l_jj.
template <int KB>
__device__ __forceinline__ void chol_warp(const double* src, int ld, double* dst, double* colj, double* invd,
                                          int lane, int* bad) {
  double ra[KB];
  const int i = lane < KB ? lane : KB - 1;
#pragma unroll
  for (int k = 0; k < KB; k += 2) {
    const double2 t = *reinterpret_cast<const double2*>(src + i * ld + k);
    ra[k] = t.x;
    ra[k + 1] = t.y;
  }
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    double piv = __shfl_sync(0xffffffffu, ra[j], j);
    if (!(piv > 0.0) || !(piv < 1e300)) {
      if (lane == 0) *bad = 1;
      piv = 1.0;
    }
    const double rs = rsqrt_pos(piv);  // 1 / l_jj; l_jj = piv / l_jj
    ra[j] = (lane == j) ? piv * rs : ra[j] * rs;
    if (lane < KB) colj[lane] = ra[j];
    if (lane == 0) invd[j] = rs;
    __syncwarp();
#pragma unroll
    for (int k = (j + 1) & ~1; k < KB; k += 2) {
      const double2 ck = *reinterpret_cast<const double2*>(colj + k);
      if (k > j) ra[k] = fma(-ra[j], ck.x, ra[k]);
      ra[k + 1] = fma(-ra[j], ck.y, ra[k + 1]);
    }
    __syncwarp();
  }
  if (lane < KB) {
#pragma unroll
    for (int k = 0; k < KB; ++k) dst[lane * ld + k] = k <= lane ? ra[k] : 0.0;
  }
  __syncwarp();
}
template <int K>
struct SubTc {
  static constexpr int LDV = K + (20 - K % 16) % 16;  // = 4 (mod 16)
  static constexpr int NT = K / 8;                     // 8-column tiles
  static constexpr size_t SMEM = ((size_t)2 * kTcD * LDV + 2 * (size_t)K * LDV + 32 + K) * sizeof(double);
};
}  // namespace

template <int K>
__global__ void __launch_bounds__(kSubThreads, K <= 32 ? 2 : 1) subspace_tc_kernel(int iters, double eps,
                                                                     const double* __restrict__ cq,
                                                                     const double* __restrict__ mu,
                                                                     const float* __restrict__ V0, bool center,
                                                                     float* __restrict__ R, float* __restrict__ dmu,
                                                                     float* __restrict__ ritz,
                                                                     int32_t* __restrict__ info) {
  using S = SubTc<K>;
  constexpr int d = kTcD, LDV = S::LDV, NT = S::NT;
  extern __shared__ __align__(16) double ssm[];
  double* V = ssm;             // [d][LDV]
  double* W = V + d * LDV;     // [d][LDV]   C V
  double* G = W + d * LDV;     // [K][LDV]
  double* L = G + K * LDV;     // [K][LDV]   lower Cholesky factor
  double* red = L + K * LDV;   // [32 + K]
  __shared__ int s_bad;
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const double* C = cq + (size_t)u * d * d;
  if (tid == 0) s_bad = 0;
  for (int e = tid; e < d * K; e += kSubThreads) V[(e / K) * LDV + e % K] = (double)V0[(size_t)u * d * K + e];
  __syncthreads();

  // W = C V: warp w, rows [16w, 16w + 16) (two 8-row tiles) x all K columns
  auto mul_CV = [&]() {
    double acc[2][NT][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const double* Crow0 = C + (size_t)(16 * warp + g) * d + c;
    const double* Crow1 = Crow0 + 8 * d;
#pragma unroll 8
    for (int k0 = 0; k0 < d; k0 += 4) {
      const double a0 = __ldg(Crow0 + k0), a1 = __ldg(Crow1 + k0);
      const double* Vk = V + (k0 + c) * LDV + g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double b = Vk[8 * nt];
        dmma(acc[0][nt], a0, b);
        dmma(acc[1][nt], a1, b);
      }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<double2*>(W + (16 * warp + 8 * mt + g) * LDV + 8 * nt + 2 * c) =
            make_double2(acc[mt][nt][0], acc[mt][nt][1]);
  };

  for (int it = 0; it < iters; ++it) {
    mul_CV();
    __syncthreads();
    // G = W^T W: 8x8 tiles (mt, nt), mt <= nt needed (the Cholesky reads the lower triangle
    // through G[j][i], i >= j... both triangles are written for simplicity)
    for (int t = warp; t < NT * NT; t += kSubThreads / 32) {
      const int mt = t / NT, nt = t % NT;
      double acc[2] = {0.0, 0.0};
#pragma unroll 8
      for (int k0 = 0; k0 < d; k0 += 4) {
        const double* Wk = W + (k0 + c) * LDV + g;
        dmma(acc, Wk[8 * mt], Wk[8 * nt]);
      }
      *reinterpret_cast<double2*>(G + (8 * mt + g) * LDV + 8 * nt + 2 * c) = make_double2(acc[0], acc[1]);
    }
    __syncthreads();
    // rho = eps tr(G) / k ; L = chol(G + rho I)
    // warp 0: rho = eps tr(G) / k, then L = chol(G + rho I) in registers -- for K = 64 blocked:
    // L11 = chol(G11); L21 = G21 L11^{-T} (row-wise substitution); L22 = chol(G22 - L21 L21^T)
    if (warp == 0) {
      double* colj = red;       // [32] current column of L
      double* invd = red + 32;  // [K] 1 / l_jj (the substitution multiplies by it)
      double tr = 0.0;
      for (int a = lane; a < K; a += 32) tr += G[a * LDV + a];
      tr = warp_sum(tr);
      const double rho = eps * tr / (double)K;
      for (int a = lane; a < K; a += 32) G[a * LDV + a] += rho;
      __syncwarp();
      if constexpr (K <= 32) {
        chol_warp<K>(G, LDV, L, colj, invd, lane, &s_bad);
      } else {
        static_assert(K == 64, "blocked Cholesky for K = 64");
        chol_warp<32>(G, LDV, L, colj, invd, lane, &s_bad);
        {  // L21: row 32 + lane solves x L11^T = G21[lane]
          double x[32];
          const double* Gr = G + (32 + lane) * LDV;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            double s0 = Gr[j], s1 = 0.0;
            const double* Lj = L + j * LDV;
#pragma unroll
            for (int m = 0; m + 1 < j; m += 2) {
              s0 = fma(-x[m], Lj[m], s0);
              s1 = fma(-x[m + 1], Lj[m + 1], s1);
            }
            if (j & 1) s0 = fma(-x[j - 1], Lj[j - 1], s0);
            x[j] = (s0 + s1) * invd[j];
          }
          double* Lr = L + (32 + lane) * LDV;
#pragma unroll
          for (int j = 0; j < 32; ++j) Lr[j] = x[j];
        }
        __syncwarp();
        {  // G22 <- G22 - L21 L21^T (lane = row 32 + lane, all 32 columns; upper part unused)
          double* Gr = G + (32 + lane) * LDV + 32;
          const double* Li = L + (32 + lane) * LDV;
          for (int k = 0; k < 32; ++k) {
            const double* Lk = L + (32 + k) * LDV;
            double s0 = Gr[k], s1 = 0.0;
#pragma unroll
            for (int m = 0; m < 32; m += 2) {
              s0 = fma(-Li[m], Lk[m], s0);
              s1 = fma(-Li[m + 1], Lk[m + 1], s1);
            }
            Gr[k] = s0 + s1;
          }
        }
        __syncwarp();
        chol_warp<32>(G + 32 * LDV + 32, LDV, L + 32 * LDV + 32, colj, invd + 32, lane, &s_bad);
        for (int k = 32; k < 64; ++k) L[lane * LDV + k] = 0.0;  // upper-right block
      }
    }
    __syncthreads();
    // V = W L^{-T}: every row x solves x L^T = w (forward substitution), the row in registers,
    // L read as shared-memory broadcasts
    if (tid < d) {
      double v[K];
      const double* Wr = W + tid * LDV;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        double s0 = Wr[j], s1 = 0.0;
        const double* Lj = L + j * LDV;
#pragma unroll
        for (int m = 0; m + 1 < j; m += 2) {
          s0 = fma(-v[m], Lj[m], s0);
          s1 = fma(-v[m + 1], Lj[m + 1], s1);
        }
        if (j & 1) s0 = fma(-v[j - 1], Lj[j - 1], s0);
        v[j] = (s0 + s1) * red[32 + j];
      }
      double* Vr = V + tid * LDV;
#pragma unroll
      for (int j = 0; j < K; ++j) Vr[j] = v[j];
    }
    __syncthreads();
  }
  // store R = V rounded to fp32; delta_mu from the stored values (fp64)
  float* Ru = R + (size_t)u * d * K;
  for (int e = tid; e < d * K; e += kSubThreads) {
    const float v = (float)V[(e / K) * LDV + e % K];
    Ru[e] = v;
    V[(e / K) * LDV + e % K] = (double)v;
  }
  __syncthreads();
  if (tid < K) {
    double s = 0.0;
    if (center)
      for (int x = 0; x < d; ++x) s = fma(V[x * LDV + tid], mu[(size_t)u * d + x], s);
    red[tid] = s;
  }
  __syncthreads();
  for (int x = tid; x < d; x += kSubThreads) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = fma(V[x * LDV + k], red[k], s);
    dmu[(size_t)u * d + x] = center ? (float)(mu[(size_t)u * d + x] - s) : 0.f;
  }
  // Rayleigh quotients of the returned basis: ritz_j = R_j^T C R_j / R_j^T R_j
  if (ritz) {
    __syncthreads();
    mul_CV();
    __syncthreads();
    for (int j = tid; j < K; j += kSubThreads) {
      double num = 0.0, den = 0.0;
      for (int i = 0; i < d; ++i) {
        num = fma(V[i * LDV + j], W[i * LDV + j], num);
        den = fma(V[i * LDV + j], V[i * LDV + j], den);
      }
      ritz[(size_t)u * K + j] = (float)(num / den);
    }
  }
  if (tid == 0 && info) info[u] = s_bad ? -1 : 0;
}

int launch_subspace(int U, int d, int k, int iters, double eps, bool center, const CalibWs& ws,
                    const float* V0, float* R, float* dmu, float* ritz, int32_t* info, cudaStream_t st) {
  if (d == kTcD && k % 8 == 0 && k <= 64) {
    switch (k) {
#define RK_SUBTC_CASE(KK)                                                                                  \
  case KK: {                                                                                               \
    const int smt = (int)SubTc<KK>::SMEM;                                                                  \
    cudaFuncSetAttribute(subspace_tc_kernel<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smt);        \
    subspace_tc_kernel<KK><<<U, kSubThreads, smt, st>>>(iters, eps, ws.cq, ws.mu, V0, center, R, dmu, ritz, \
                                                        info);                                             \
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;                                                  \
  }
      RK_SUBTC_CASE(8)
      RK_SUBTC_CASE(16)
      RK_SUBTC_CASE(32)
      RK_SUBTC_CASE(64)
#undef RK_SUBTC_CASE
    }
  }
  const size_t sm = subspace_smem_bytes(d, k);
  if (sm > 227 * 1024) return -2;
  switch (k) {
#define RK_SUB_CASE(KK)                                                                                    \
  case KK:                                                                                                 \
    cudaFuncSetAttribute(subspace_kernel<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);       \
    subspace_kernel<KK><<<U, kSubThreads, sm, st>>>(d, iters, eps, ws.cq, ws.mu, V0, center, R, dmu, ritz, \
                                                    info);                                                 \
    break;
    RK_SUB_CASE(4)
    RK_SUB_CASE(8)
    RK_SUB_CASE(16)
    RK_SUB_CASE(32)
    RK_SUB_CASE(64)
#undef RK_SUB_CASE
    default:
      return -2;
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rk
