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

int launch_subspace(int U, int d, int k, int iters, double eps, bool center, const CalibWs& ws,
                    const float* V0, float* R, float* dmu, float* ritz, int32_t* info, cudaStream_t st) {
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
