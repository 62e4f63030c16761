// tok_gather.cuh -- token selection fused into the prefill producers (NEXT-2).
//
// The tensor-core covariance (cov_tc.cu) and compress (compress_tc.cu) kernels normally load a
// 128-token x 128-channel key tile with two tensor-map TMA boxes (64-channel halves, 128-byte
// swizzle).  With a token list (FastV / VisionZip survivors: unit u keeps rows tok_idx[u][t] of
// its n_src-row key block) or per-unit valid lengths (a padded batch of requests with different
// image-token counts), the producer warp instead gathers the tile itself: every lane issues
// 16-byte cp.async copies of its rows straight into the SAME swizzled layout, and rows past the
// unit's valid count (or with an out-of-range index) are zero-filled without reading memory
// (src-size 0).  So the survivors are never compacted by a separate read+write pass, and
// padding never reaches C_q or K~.  Completion: each lane's copies are tracked by
// cp.async.mbarrier.arrive.noinc on the stage's `full` barrier (initialised with 32 arrivals);
// the MMA thread fences the async proxy after its wait (generic-proxy writes -> tcgen05 reads).
#pragma once

#include "common.cuh"

namespace rk {

struct TokSrc {
  const int32_t* idx = nullptr;  // [U][n_log] row of K[u] for logical token t (or null: t itself)
  const int32_t* nvu = nullptr;  // [U] valid logical tokens (or null: n_log)
  int n_src = 0;                 // rows per unit of K (== n_log without idx)
  __host__ __device__ bool active() const { return idx != nullptr || nvu != nullptr; }
  __device__ __forceinline__ int valid(int u, int n_log) const {
    if (nvu == nullptr) return n_log;
    const int v = __ldg(nvu + u);
    return v < 0 ? 0 : (v < n_log ? v : n_log);
  }
};

__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// arrive on `bar` when all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Fill one stage with logical tokens [tok0, tok0 + 128) of unit u: two 64-channel halves of
// [128 rows][128 B], 16-byte chunk c of row t at t * 128 + ((c ^ (t & 7)) << 4) (the 128-byte
// swizzle TMA produces).  One warp; each instruction covers two tokens' 512 contiguous bytes.
__device__ __forceinline__ void gather_tile_128x128(const TokSrc& src, const __nv_bfloat16* K, int u, int n_log,
                                                    int nv, int tok0, unsigned char* stage, int half_bytes,
                                                    int lane) {
  const uint32_t sbase = smem_u32(stage);
#pragma unroll 4
  for (int i = lane; i < 128 * 16; i += 32) {
    const int t = i >> 4, pc = i & 15;
    const int tl = tok0 + t;
    int row = tl;
    bool ok = tl < nv;
    if (ok && src.idx != nullptr) {
      row = __ldg(src.idx + (size_t)u * n_log + tl);
      ok = row >= 0 && row < src.n_src;
    }
    const char* g = reinterpret_cast<const char*>(K + ((size_t)u * src.n_src + (ok ? row : 0)) * 128) + pc * 16;
    const uint32_t dst = sbase + (pc >> 3) * half_bytes + t * 128 + (((pc & 7) ^ (t & 7)) << 4);
    cp_async_16(dst, g, ok ? 16u : 0u);
  }
}

}  // namespace rk
