// decode_common.cuh -- declarations shared by the decode translation units (decode.cu: the
// generic, CUDA-core streaming, per-warp GQA and work-stealing kernels; decode_ring.cu: the
// CTA-ring GQA kernel).  Device code only plus two host launch helpers.
#pragma once

#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace rk {

struct DecodeParams {
  int U, G, d, r, N, M;
  const void* q;
  const void* Kc;
  const void* V;
  const float* R;
  const float* dmu;
  const void* Kt;
  const void* Vt;
  float sl;  // softmax scale * log2(e)
  float* out;
  uint32_t* counters;
  float* partials;
  unsigned long long* trace = nullptr;  // diagnostics: [NW][8] globaltimer stamps (or null)
  int aw = 0;                           // active (streaming) warps per CTA (<= WARPS)
  float* pout = nullptr;                // partial-state output [U][G][d+2] (token shards) or null
  int nR = 0;                           // unit u uses R[u % nR], dmu[u % nR]
  unsigned long long* desc = nullptr;   // work stealing: per-warp range descriptors
  uint32_t* nslot = nullptr;            // work stealing: partial slots per unit
  int overlap = 0;                      // programmatic dependent launch (ROTATEK_DECODE_OVERLAP)
  int Ms = 0;                           // K_text / V_text rows per unit (text_stride)
  const int32_t* nvu = nullptr;         // variable lengths: valid visual tokens per unit (or null)
  const int32_t* ntu = nullptr;         // variable lengths: valid text tokens per unit (or null)
};

// tokens of tile (u, vis, t, tn) that lie inside the unit's valid length (variable-length
// units over padded caches; every token when no lengths are given)
__device__ __forceinline__ int valid_tn(const DecodeParams& p, int u, bool vis, int t, int tn) {
  const int32_t* lens = vis ? p.nvu : p.ntu;
  if (lens == nullptr) return tn;
  const int v = __ldg(lens + u) - t;
  return v <= 0 ? 0 : (v < tn ? v : tn);
}

// Programmatic dependent launch.  Every streaming decode lets the next kernel on the stream
// launch early (it must then griddepcontrol.wait before reading out); with `overlap` the
// decode itself was launched early and waits before its first read of q / workspace.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int kD = 128;

// Per-unit query table entry (see rotate_unit): qt [G][RK] f32 | b [G] f32 (16-B padded) |
// q [G][kD] in the cache dtype.
template <typename T, int RK, int G>
struct QEnt {
  static constexpr int OFF_B = G * RK * 4;
  static constexpr int OFF_Q = OFF_B + ((G + 3) / 4) * 16;
  static constexpr int BYTES = (OFF_Q + G * kD * (int)sizeof(T) + 15) / 16 * 16;
};

namespace gqa {

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// element x0 -> low 16 bits, x1 -> high 16 bits
__device__ __forceinline__ uint32_t pack2(float x0, float x1) {
  __nv_bfloat162 v = __floats2bfloat162_rn(x0, x1);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack2(x0 - hf.x, x1 - hf.y);
}
// byte offset of a 16-byte chunk in a row of a swizzled TMA box (rows of RB bytes)
template <int RB>
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
  const uint32_t off = row * RB + chunk * 16;
  if constexpr (RB == 128) return off ^ (((off >> 7) & 7u) << 4);
  else return off ^ (((off >> 7) & 3u) << 4);  // RB == 64: 64-byte swizzle
}

}  // namespace gqa

// the calling thread's diagnostics buffer (rotatek_debug_decode_trace; null normally)
unsigned long long* decode_trace_buffer();
int decode_num_sms();

template <typename Kern, typename... Args>
static bool launch(Kern kern, int ctas, int threads, size_t smem, cudaStream_t st, Args... args) {
  kern<<<ctas, threads, smem, st>>>(args...);
  return cudaPeekAtLastError() == cudaSuccess;
}

// launch as a programmatic dependent of the preceding work on the stream
template <typename Kern, typename... Args>
static bool launch_overlap(Kern kern, int ctas, int threads, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...) == cudaSuccess;
}

}  // namespace rk
