// internal.h -- host-side launchers behind the C ABI (not exported).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "tok_gather.cuh"

namespace rk {

constexpr int kNumSMs = 148;
constexpr int kMaxDevices = 64;

// Once-per-(call site, device) setup: kernel attributes such as the >48 KB dynamic shared
// memory opt-in are per-device state, so a process driving several GPUs must set them on
// each.  slot[dev] caches init()'s (positive) result for the current device; a race between
// threads only repeats the idempotent init.
template <typename F>
int once_per_device(int (&slot)[kMaxDevices], F&& init) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return init();
  int v = __atomic_load_n(&slot[dev], __ATOMIC_ACQUIRE);
  if (v <= 0) {
    v = init();
    __atomic_store_n(&slot[dev], v, __ATOMIC_RELEASE);
  }
  return v;
}

struct CalibWs {
  double* sigma;     // [U, d]
  double* covpart;   // [U, P, d, d]   upper tiles valid
  double* colpart;   // [U, P, d]
  double* cq;        // [U, d, d]
  double* mu;        // [U, d]
  float* lam;        // [U, d]
  void* vecs;        // [U, d, d] double (eigenvectors, columns in solver order)
  float* v32;        // [U, d, d] fp32 Jacobi basis before the fp64 refinement
  int32_t* jinfo;    // [U]
  int parts;         // P token partitions per unit
};

struct DecodeWs {
  uint32_t* counters;  // [U] zero on entry, left zero
  float* partials;     // [U, G, S, d + 2] (generic) or [U, cmax, G, d + 4] (streaming)
  unsigned long long* desc;  // [kMaxStealWarps] work-stealing range descriptors (left exhausted)
  uint32_t* nslot;           // [U] partial slots handed out per unit (zero on entry, left zero)
  size_t partial_bytes;      // capacity of `partials`
  int max_splits;
};
constexpr int kMaxStealWarps = kNumSMs * 16;

int cov_parts(int U, int N);
int decode_max_splits(int U, int N, int M);
size_t calib_ws_layout(int U, int d, int N, bool fp64_eig, void* base, CalibWs* ws);
size_t decode_ws_layout(int U, int G, int d, int r, int N, int M, void* base, DecodeWs* ws);

// each returns the number of launches enqueued (>= 0) or -1 on launch error
int launch_sigma(int U, int G, int W, int d, bool bf16, bool weight, const void* Qw,
                 double* sigma, cudaStream_t st);
int launch_cov(int U, int N, int d, bool bf16, const void* K, const CalibWs& ws, cudaStream_t st);
bool cov_tc_supported(int d, bool bf16);
bool compress_tc_supported(int d, int r, bool bf16);
int launch_compress_tc(int U, int N, int r, const void* K, const float* R, void* Kc, cudaStream_t st,
                       int nR = 0, const TokSrc& tsrc = TokSrc());
// parts == 1 also finalizes (writes cq and mu): the caller skips launch_finalize
int launch_cov_tc(int U, int N, bool center, const void* K, const CalibWs& ws, cudaStream_t st,
                  bool allow_fused = true, const TokSrc& tsrc = TokSrc());
// calibration statistics state (rotatek_calib_accumulate / rotatek_calibrate_from_state)
int launch_state_accumulate(int U, int N, int d, int nS, bool weight, const CalibWs& ws, double* state,
                            cudaStream_t st);
int launch_state_finalize(int nS, int d, bool center, bool weight, const double* state, const CalibWs& ws,
                          cudaStream_t st);
int launch_finalize(int U, int N, int d, bool center, const CalibWs& ws, cudaStream_t st,
                    const int32_t* nvu = nullptr);
int launch_jacobi(int U, int d, int r, bool fp64, bool twosided, const CalibWs& ws, cudaStream_t st);
int launch_select_gather(int U, int d, int r, bool fp64_vecs, bool bf16x2, bool center,
                         const CalibWs& ws, float* R, float* dmu, float* eigvals,
                         uint32_t* mask, int32_t* idx, float* R_full, int32_t* info,
                         cudaStream_t st);
int launch_subspace(int U, int d, int k, int iters, double eps, bool center, const CalibWs& ws,
                    const float* V0, float* R, float* dmu, float* ritz, int32_t* info, cudaStream_t st);
int launch_select_only(int U, int d, int r, const float* lam, uint32_t* mask, int32_t* idx,
                       int32_t* info, cudaStream_t st);
int launch_gather_rows(int U, int n_src, int n_keep, int row_bytes, const int32_t* idx, const void* src,
                       void* dst, int32_t* err, cudaStream_t st);
int launch_compress(int U, int N, int d, int r, bool bf16, const void* K, const float* R,
                    void* Kc, cudaStream_t st, int nR = 0);

struct DecodeArgs {
  int U, G, d, r, N, M;
  bool bf16;
  const void* q;
  const void* Kc;
  const void* V;
  const float* R;
  const float* dmu;
  const void* Kt;
  const void* Vt;
  float scale;
  float* out;
  float* pout = nullptr;  // token-shard partial state [U][G][d+2] instead of out
  int nR = 0;             // distinct rotations: unit u uses R[u % nR], dmu[u % nR] (0: nR = U)
  int overlap = 0;        // ROTATEK_DECODE_OVERLAP: programmatic dependent launch
  int Ms = 0;             // K_text / V_text rows per unit (text_stride; >= M)
  const int32_t* nvu = nullptr;  // variable lengths (rotatek_decode_attn_varlen) or null
  const int32_t* ntu = nullptr;
};
// kernel: 0 auto, 1 generic, 2 fast.  Returns launches, -1 launch error, -2 unsupported.
int launch_merge_parts(int U, int G, int d, int P, const float* parts, float* out, cudaStream_t st);
void set_decode_trace(void* buf);  // diagnostics (rotatek_debug_decode_trace)
int launch_decode(const DecodeArgs& a, const DecodeWs& ws, int splits, int kernel,
                  cudaStream_t st);
// the CTA-ring GQA kernel (decode_ring.cu); -3: shape not served (caller falls back)
int launch_ring(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st);

}  // namespace rk
