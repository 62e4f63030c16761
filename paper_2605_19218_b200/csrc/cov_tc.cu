// cov_tc.cu -- Alg. 1 lines 1-3: the key Gram matrix S = sum_n K_n K_n^T and the
// column sums sum_n K_n, on the 5th-generation tensor cores (tcgen05) for d = 128, bf16 keys.
//
//   C = K^T K as one GEMM D[d x d] = A[d x tok] . B[tok x d] where A = K^T and B = K are the
//   SAME shared-memory tile read through two MN-major descriptors (128-byte swizzle).
//   TMA (cp.async.bulk.tensor.3d, SWIZZLE_128B) brings 128-token x 128-channel chunks into a
//   4-stage ring; one elected thread issues 8 tcgen05.mma (M=128, N=128, K=16) per chunk into
//   one of two 128-column fp32 accumulators in TMEM; eight epilogue warps drain the other
//   accumulator with tcgen05.ld and add it into fp64 registers, so each fp32 accumulation
//   spans at most 128 tokens (exact bf16 products, fp32 per chunk, fp64 across chunks: the
//   precision scheme of SURVEY Appendix A E-5/E-6).  The epilogue warps also form the column
//   sums from the staged tile.  Out-of-range tokens of the last chunk are zero-filled by TMA.
//
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2..9 epilogue (TMEM lane quadrant = warp % 4, column half = (warp - 2) / 4).
#include <cstdio>

#include "internal.h"
#include "tc_common.cuh"

namespace rk {

namespace {
constexpr int kTK = 128;                 // tokens per chunk (fp32 accumulation window)
constexpr int kDc = 128;                 // head dim
constexpr int kStages = 4;
constexpr int kHalfBytes = kTK * 128;    // one 64-channel half: kTK rows x 128 B
constexpr int kStageBytes = 2 * kHalfBytes;
constexpr int kThreads = 320;
constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
}  // namespace

__global__ void __launch_bounds__(kThreads, 1) cov_tc_kernel(const __grid_constant__ CUtensorMap tmap, int N,
                                                             int parts, double* __restrict__ covpart,
                                                             double* __restrict__ colpart) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ double colred[2][kDc];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.y, p = blockIdx.x;
  const int nchunks_all = (N + kTK - 1) / kTK;
  const int c_lo = (int)((long long)nchunks_all * p / parts);
  const int c_hi = (int)((long long)nchunks_all * (p + 1) / parts);
  const int nch = c_hi - c_lo;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 8);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_mbar_init();
    tc::prefetch_tmap(&tmap);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < nch; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        unsigned char* dst = sm + s * kStageBytes;
        mbar_arrive_expect_tx(&full[s], kStageBytes);
        const int tok = (c_lo + i) * kTK;
        tc::tma_load_3d(dst, &tmap, 0, tok, u, &full[s], pol);
        tc::tma_load_3d(dst + kHalfBytes, &tmap, 64, tok, u, &full[s], pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, 128, true, true);
      for (int i = 0; i < nch; ++i) {
        const int s = i % kStages, a = i & 1;
        mbar_wait(&full[s], (i / kStages) & 1);
        mbar_wait(&tempty[a], ((i >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t base = smem_u32(sm + s * kStageBytes);
#pragma unroll
        for (int kk = 0; kk < kTK / 16; ++kk) {
          // MN-major, SWIZZLE_128B: LBO = next 64-channel half, SBO = next 8-token group
          const uint64_t desc = tc::smem_desc(base + kk * 16 * 128, kHalfBytes, 1024, tc::SWZ_128B);
          tc::mma_bf16(tmem + a * 128, desc, desc, idesc, kk > 0 ? 1u : 0u);
        }
        tc::commit(&empty[s]);
        tc::commit(&tfull[a]);
      }
    }
  } else {
    // ---------------- epilogue: 8 warps
    const int e = warp - 2;
    const int q = warp & 3;        // TMEM lane quadrant this warp may access
    const int h = e >> 2;          // accumulator column half
    const int row = 32 * q + lane;  // output row (channel i)
    const int cch = (e * 32 + lane) & (kDc - 1);  // colsum channel
    const int thalf = (e * 32 + lane) >> 7;       // colsum token half (0..1)
    double acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0;
    double csum = 0.0;
    for (int i = 0; i < nch; ++i) {
      const int s = i % kStages, a = i & 1;
      // column sums from the staged (swizzled) tile
      mbar_wait(&full[s], (i / kStages) & 1);
      {
        const unsigned char* half = sm + s * kStageBytes + (cch >> 6) * kHalfBytes;
        const int c64 = cch & 63, chunk = c64 >> 3, within = (c64 & 7) * 2;
        float fs = 0.f;
#pragma unroll 8
        for (int t = 0; t < 64; ++t) {
          const int n = thalf * 64 + t;
          const uint16_t v = *reinterpret_cast<const uint16_t*>(half + n * 128 + ((chunk ^ (n & 7)) << 4) + within);
          fs += __uint_as_float((uint32_t)v << 16);
        }
        csum += (double)fs;
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[s]);
      // drain the accumulator of this chunk into fp64
      mbar_wait(&tfull[a], (i >> 1) & 1);
      tc::fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + a * 128 + h * 64;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        uint32_t r[16];
        tc::ld_32x32b_x16(taddr + b * 16, r);
        tc::ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[b * 16 + j] += (double)__uint_as_float(r[j]);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[a]);
    }
    double* out = covpart + ((size_t)u * parts + p) * kDc * kDc + (size_t)row * kDc + h * 64;
#pragma unroll
    for (int j = 0; j < 64; j += 2) *reinterpret_cast<double2*>(out + j) = make_double2(acc[j], acc[j + 1]);
    colred[thalf][cch] = csum;
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < kDc)
    colpart[((size_t)u * parts + p) * kDc + threadIdx.x] = colred[0][threadIdx.x] + colred[1][threadIdx.x];
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 256);
  }
}

// ------------------------------------------------------------------------------ host
using PFN_encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encode get_encode() {
  static PFN_encode fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_encode>(p);
  }();
  return fn;
}

bool encode_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                         uint32_t b1, int swizzle_bytes) {
  PFN_encode enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool cov_tc_supported(int d, bool bf16) { return bf16 && d == kDc && get_encode() != nullptr; }

int launch_cov_tc(int U, int N, const void* K, const CalibWs& ws, cudaStream_t st) {
  CUtensorMap map;
  if (!encode_tmap_3d_bf16(&map, K, kDc, (uint64_t)N, (uint64_t)U, 64, kTK, 128)) return -2;
  static bool attr = [] {
    return cudaFuncSetAttribute(cov_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) == cudaSuccess;
  }();
  (void)attr;
  dim3 grid(ws.parts, U);
  cov_tc_kernel<<<grid, kThreads, kSmem, st>>>(map, N, ws.parts, ws.covpart, ws.colpart);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rk
