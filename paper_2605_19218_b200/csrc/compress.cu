// compress.cu -- Alg. 1 line 14: K~ = K R_r, stored in place of K,
// rounded (RNE) to the cache dtype.  R_r is the stored calibrate output (bf16 path: every
// value is exactly bf16_hi + bf16_lo), used identically by decode for q~ (reading E-11).
//
// v1: CUDA-core fp32 FMA.  One CTA per (64-token tile, unit); R_r [d, r] and the K tile
// [64, d] are staged in shared memory as fp32; each warp owns 8 tokens, each lane a
// strided set of output channels.
#include "common.cuh"
#include "internal.h"

namespace rk {

constexpr int kCmpTok = 64;

template <typename T>
__global__ void __launch_bounds__(256) compress_kernel(int N, int d, int r, const T* __restrict__ K,
                                                       const float* __restrict__ R,
                                                       T* __restrict__ Kc, int nR) {
  extern __shared__ __align__(16) float csm[];
  float* Rs = csm;               // [d][r]
  float* Ks = csm + d * r;       // [kCmpTok][d]
  const int u = blockIdx.y, t0 = blockIdx.x * kCmpTok;
  const int tn = min(kCmpTok, N - t0);
  const int tid = threadIdx.x;
  const float* Ru = R + (size_t)(u % nR) * d * r;  // nR < U: a shared (offline) rotation
  for (int e = tid; e < d * r; e += blockDim.x) Rs[e] = Ru[e];
  const T* Ku = K + ((size_t)u * N + t0) * d;
  for (int e = tid; e < tn * d; e += blockDim.x) Ks[e] = Elem<T>::to_f(Ku[e]);
  __syncthreads();
  const int w = tid >> 5, lane = tid & 31;
  T* out = Kc + ((size_t)u * N + t0) * r;
  for (int k = lane; k < r; k += 32) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int i = 0; i < d; ++i) {
      const float rv = Rs[i * r + k];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fmaf(Ks[(w * 8 + j) * d + i], rv, acc[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = w * 8 + j;
      if (t < tn) out[(size_t)t * r + k] = Elem<T>::from_f(acc[j]);
    }
  }
}

int launch_compress(int U, int N, int d, int r, bool bf16, const void* K, const float* R,
                    void* Kc, cudaStream_t st, int nR) {
  if (nR <= 0) nR = U;
  dim3 grid((N + kCmpTok - 1) / kCmpTok, U);
  size_t sm = ((size_t)d * r + (size_t)kCmpTok * d) * sizeof(float);
  if (bf16) {
    cudaFuncSetAttribute(compress_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    compress_kernel<__nv_bfloat16><<<grid, 256, sm, st>>>(N, d, r, (const __nv_bfloat16*)K, R,
                                                         (__nv_bfloat16*)Kc, nR);
  } else {
    cudaFuncSetAttribute(compress_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    compress_kernel<float><<<grid, 256, sm, st>>>(N, d, r, (const float*)K, R, (float*)Kc, nR);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ============================================================== token gather (NEXT-2)
// dst[u][j] = src[u][idx[u][j]] for row bytes `rb` (token pruning: FastV / VisionZip
// keep a scattered subset of visual tokens; calibrate, compress and decode then run on the
// compacted cache).  One warp per destination row, 16-byte vectors; out-of-range indices
// set *err (the rows are zero-filled).
__global__ void __launch_bounds__(256) gather_rows_kernel(int U, int n_src, int n_keep, int rb16,
                                                          const int32_t* __restrict__ idx,
                                                          const uint4* __restrict__ src,
                                                          uint4* __restrict__ dst, int32_t* __restrict__ err) {
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long long)U * n_keep) return;
  const int u = (int)(row / n_keep);
  const int t = __ldg(idx + row);
  uint4* d = dst + row * rb16;
  if (t < 0 || t >= n_src) {
    for (int e = lane; e < rb16; e += 32) d[e] = make_uint4(0u, 0u, 0u, 0u);
    if (lane == 0 && err) atomicExch(err, 1);
    return;
  }
  const uint4* s = src + ((long long)u * n_src + t) * rb16;
  for (int e = lane; e < rb16; e += 32) d[e] = __ldcs(s + e);
}

int launch_gather_rows(int U, int n_src, int n_keep, int row_bytes, const int32_t* idx, const void* src,
                       void* dst, int32_t* err, cudaStream_t st) {
  const long long rows = (long long)U * n_keep;
  gather_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(U, n_src, n_keep, row_bytes / 16, idx,
                                                                 static_cast<const uint4*>(src),
                                                                 static_cast<uint4*>(dst), err);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rk
