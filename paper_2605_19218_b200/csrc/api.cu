// api.cu -- the C ABI of librotatek.so (declared in include/rotatek.h).
// Host-side validation, workspace carving and kernel launches; never synchronises.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/rotatek.h"
#include "internal.h"

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

rotatek_status fail(rotatek_status s, const char* fmt, const char* what = "") {
  snprintf(g_err, sizeof(g_err), fmt, what);
  return s;
}

// every entry point starts here: reset the launch count and clear a stale (non-sticky)
// runtime error left by the caller's earlier CUDA calls, so the per-launch checks
// (cudaPeekAtLastError) only ever see this call's own launches
void begin_call() {
  g_launches = 0;
  (void)cudaGetLastError();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

rotatek_status check_dims(const rotatek_dims* dm) {
  if (!dm) return fail(ROTATEK_ERR_NULL, "dims is NULL");
  if (dm->units < 1) return fail(ROTATEK_ERR_DIMS, "units must be >= 1");
  if (dm->group < 1) return fail(ROTATEK_ERR_DIMS, "group must be >= 1");
  if (dm->head_dim < 16 || dm->head_dim > 256 || dm->head_dim % 16 != 0)
    return fail(ROTATEK_ERR_DIMS, "head_dim must be a multiple of 16 in [16, 256]");
  if (dm->rank < 1 || dm->rank > dm->head_dim) return fail(ROTATEK_ERR_DIMS, "rank must be in [1, head_dim]");
  if (dm->n_vis < 1) return fail(ROTATEK_ERR_DIMS, "n_vis must be >= 1 (empty visual segment)");
  if (dm->n_text < 0) return fail(ROTATEK_ERR_DIMS, "n_text must be >= 0");
  if (dm->q_window < 0) return fail(ROTATEK_ERR_DIMS, "q_window must be >= 0");
  if (dm->dtype != ROTATEK_BF16 && dm->dtype != ROTATEK_F32) return fail(ROTATEK_ERR_DIMS, "bad dtype");
  if (dm->text_stride < 0 || (dm->text_stride > 0 && dm->text_stride < dm->n_text))
    return fail(ROTATEK_ERR_DIMS, "text_stride must be 0 or >= n_text");
  return ROTATEK_OK;
}

rotatek_status launched(int rc, int* count) {
  if (rc == -2) return fail(ROTATEK_ERR_UNSUPPORTED, "no kernel for this shape");
  if (rc < 0) {
    cudaError_t e = cudaGetLastError();
    return fail(ROTATEK_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
  }
  *count += rc;
  return ROTATEK_OK;
}

}  // namespace

extern "C" {

int rotatek_abi_version(void) { return ROTATEK_ABI_VERSION; }
const char* rotatek_last_error(void) { return g_err; }
int rotatek_last_launch_count(void) { return g_launches; }
void rotatek_debug_decode_trace(void* buf) { rk::set_decode_trace(buf); }

const char* rotatek_status_string(rotatek_status s) {
  switch (s) {
    case ROTATEK_OK: return "ROTATEK_OK";
    case ROTATEK_ERR_NULL: return "ROTATEK_ERR_NULL";
    case ROTATEK_ERR_DIMS: return "ROTATEK_ERR_DIMS";
    case ROTATEK_ERR_ALIGN: return "ROTATEK_ERR_ALIGN";
    case ROTATEK_ERR_WORKSPACE: return "ROTATEK_ERR_WORKSPACE";
    case ROTATEK_ERR_UNSUPPORTED: return "ROTATEK_ERR_UNSUPPORTED";
    case ROTATEK_ERR_CUDA: return "ROTATEK_ERR_CUDA";
  }
  return "ROTATEK_ERR_UNKNOWN";
}

size_t rotatek_workspace_bytes(const rotatek_dims* dm, rotatek_op op) {
  if (check_dims(dm) != ROTATEK_OK) return 0;
  if (op == ROTATEK_OP_CALIBRATE)
    return rk::calib_ws_layout(dm->units, dm->head_dim, dm->n_vis, true, nullptr, nullptr);
  if (op == ROTATEK_OP_DECODE)
    return rk::decode_ws_layout(dm->units, dm->group, dm->head_dim, dm->rank, dm->n_vis, dm->n_text, nullptr,
                                nullptr);
  return 0;
}

namespace {
// rotatek_calibrate / rotatek_calibrate_tokens (tsrc: token list or per-unit lengths)
rotatek_status calibrate_impl(const rotatek_dims* dm, uint32_t flags, const void* K, const rk::TokSrc& tsrc,
                              const void* Qw, float* R, float* dmu, float* eigvals, uint32_t* keep_mask,
                              int32_t* keep_idx, float* R_full, int32_t* info, void* workspace,
                              size_t workspace_bytes, rotatek_stream_t stream) {
  rotatek_status s = check_dims(dm);
  if (s != ROTATEK_OK) return s;
  const int U = dm->units, G = dm->group, d = dm->head_dim, r = dm->rank, N = dm->n_vis,
            W = dm->q_window;
  const bool bf16 = dm->dtype == ROTATEK_BF16;
  const bool weight = (flags & ROTATEK_QUERY_WEIGHT) && W > 0;
  const bool center = (flags & ROTATEK_CENTER) != 0;
  const bool fp64 = !bf16 || (flags & ROTATEK_EIG_FP64);
  if (!K || !R || !dmu) return fail(ROTATEK_ERR_NULL, "K, R and dmu are required");
  if (W > 0 && !Qw) return fail(ROTATEK_ERR_DIMS, "Qw is NULL but q_window > 0");
  if (d > 128) return fail(ROTATEK_ERR_UNSUPPORTED, "calibrate supports head_dim <= 128");
  const void* ptrs[] = {K, Qw, R, dmu, eigvals, keep_mask, keep_idx, R_full, info, workspace};
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  rk::CalibWs ws;
  const size_t need = rk::calib_ws_layout(U, d, N, true, workspace, &ws);
  if (!workspace || workspace_bytes < need) return fail(ROTATEK_ERR_WORKSPACE, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int n = 0;
  const bool tc = !(flags & ROTATEK_SIMT_ONLY) && rk::cov_tc_supported(d, bf16);
  if (tsrc.active() && !tc)
    return fail(ROTATEK_ERR_UNSUPPORTED, "token lists / per-unit lengths need the tensor-core path (bf16, d = 128)");
  if ((s = launched(rk::launch_sigma(U, G, W, d, bf16, weight, Qw, ws.sigma, st), &n))) return s;
  if ((s = launched(tc ? rk::launch_cov_tc(U, N, center, K, ws, st, true, tsrc)
                       : rk::launch_cov(U, N, d, bf16, K, ws, st),
                    &n)))
    return s;
  if (!(tc && ws.parts == 1))  // the tensor-core kernel finalizes in place when one CTA sees the unit
    if ((s = launched(rk::launch_finalize(U, N, d, center, ws, st, tsrc.nvu), &n))) return s;
  if ((s = launched(rk::launch_jacobi(U, d, r, fp64, (flags & ROTATEK_EIG_TWOSIDED) != 0, ws, st), &n))) return s;
  if ((s = launched(rk::launch_select_gather(U, d, r, /*fp64_vecs=*/true, bf16, center, ws, R, dmu, eigvals,
                                             keep_mask, keep_idx, R_full, info, st), &n)))
    return s;
  g_launches = n;
  return ROTATEK_OK;
}
}  // namespace

rotatek_status rotatek_calibrate(const rotatek_dims* dm, uint32_t flags, const void* K,
                                 const void* Qw, float* R, float* dmu, float* eigvals,
                                 uint32_t* keep_mask, int32_t* keep_idx, float* R_full,
                                 int32_t* info, void* workspace, size_t workspace_bytes,
                                 rotatek_stream_t stream) {
  begin_call();
  return calibrate_impl(dm, flags, K, rk::TokSrc(), Qw, R, dmu, eigvals, keep_mask, keep_idx, R_full, info,
                        workspace, workspace_bytes, stream);
}

rotatek_status rotatek_calibrate_tokens(const rotatek_dims* dm, uint32_t flags, const void* K, int32_t n_src,
                                        const int32_t* tok_idx, const int32_t* n_vis_u, const void* Qw,
                                        float* R, float* dmu, float* eigvals, uint32_t* keep_mask,
                                        int32_t* keep_idx, float* R_full, int32_t* info, void* workspace,
                                        size_t workspace_bytes, rotatek_stream_t stream) {
  begin_call();
  if ((tok_idx && !aligned16(tok_idx)) || (n_vis_u && !aligned16(n_vis_u)))
    return fail(ROTATEK_ERR_ALIGN, "token arrays not 16-byte aligned");
  if (tok_idx && n_src < 1) return fail(ROTATEK_ERR_DIMS, "n_src must be >= 1 with a token list");
  rk::TokSrc tsrc;
  tsrc.idx = tok_idx;
  tsrc.nvu = n_vis_u;
  tsrc.n_src = tok_idx ? n_src : (dm ? dm->n_vis : 0);
  return calibrate_impl(dm, flags, K, tsrc, Qw, R, dmu, eigvals, keep_mask, keep_idx, R_full, info,
                        workspace, workspace_bytes, stream);
}

rotatek_status rotatek_calibrate_subspace(const rotatek_dims* dm, uint32_t flags, const void* K,
                                          const void* Qw, const float* V0, int32_t iters,
                                          float ridge, float* R, float* dmu, float* ritz,
                                          int32_t* info, void* workspace, size_t workspace_bytes,
                                          rotatek_stream_t stream) {
  begin_call();
  rotatek_status s = check_dims(dm);
  if (s != ROTATEK_OK) return s;
  const int U = dm->units, G = dm->group, d = dm->head_dim, r = dm->rank, N = dm->n_vis,
            W = dm->q_window;
  const bool bf16 = dm->dtype == ROTATEK_BF16;
  const bool weight = (flags & ROTATEK_QUERY_WEIGHT) && W > 0;
  const bool center = (flags & ROTATEK_CENTER) != 0;
  if (!K || !V0 || !R || !dmu) return fail(ROTATEK_ERR_NULL, "K, V0, R and dmu are required");
  if (W > 0 && !Qw) return fail(ROTATEK_ERR_DIMS, "Qw is NULL but q_window > 0");
  if (d > 128 || !(r == 4 || r == 8 || r == 16 || r == 32 || r == 64))
    return fail(ROTATEK_ERR_UNSUPPORTED, "subspace solver: head_dim <= 128, rank in {4,8,16,32,64}");
  const void* ptrs[] = {K, Qw, V0, R, dmu, ritz, info, workspace};
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  rk::CalibWs ws;
  const size_t need = rk::calib_ws_layout(U, d, N, true, workspace, &ws);
  if (!workspace || workspace_bytes < need) return fail(ROTATEK_ERR_WORKSPACE, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int T = iters > 0 ? iters : 5;
  const double eps = ridge >= 0.f ? (double)ridge : 1e-6;
  int n = 0;
  if ((s = launched(rk::launch_sigma(U, G, W, d, bf16, weight, Qw, ws.sigma, st), &n))) return s;
  const bool tc = !(flags & ROTATEK_SIMT_ONLY) && rk::cov_tc_supported(d, bf16);
  if ((s = launched(tc ? rk::launch_cov_tc(U, N, center, K, ws, st) : rk::launch_cov(U, N, d, bf16, K, ws, st),
                    &n)))
    return s;
  if (!(tc && ws.parts == 1))  // the tensor-core kernel finalizes in place when one CTA sees the unit
    if ((s = launched(rk::launch_finalize(U, N, d, center, ws, st), &n))) return s;
  if ((s = launched(rk::launch_subspace(U, d, r, T, eps, center, ws, V0, R, dmu, ritz, info, st), &n)))
    return s;
  g_launches = n;
  return ROTATEK_OK;
}

rotatek_status rotatek_calib_accumulate(const rotatek_dims* dm, uint32_t flags, const void* K,
                                        const void* Qw, int32_t state_units, double* state,
                                        void* workspace, size_t workspace_bytes, rotatek_stream_t stream) {
  begin_call();
  rotatek_status s = check_dims(dm);
  if (s != ROTATEK_OK) return s;
  const int U = dm->units, G = dm->group, d = dm->head_dim, N = dm->n_vis, W = dm->q_window;
  const bool bf16 = dm->dtype == ROTATEK_BF16;
  const bool weight = (flags & ROTATEK_QUERY_WEIGHT) && W > 0;
  if (!K || !state) return fail(ROTATEK_ERR_NULL, "K and state are required");
  if (W > 0 && !Qw) return fail(ROTATEK_ERR_DIMS, "Qw is NULL but q_window > 0");
  if (state_units < 1 || U % state_units != 0) return fail(ROTATEK_ERR_DIMS, "state_units must divide units");
  if (d > 128) return fail(ROTATEK_ERR_UNSUPPORTED, "calibrate supports head_dim <= 128");
  const void* ptrs[] = {K, Qw, state, workspace};
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  rk::CalibWs ws;
  const size_t need = rk::calib_ws_layout(U, d, N, true, workspace, &ws);
  if (!workspace || workspace_bytes < need) return fail(ROTATEK_ERR_WORKSPACE, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int n = 0;
  if ((s = launched(rk::launch_sigma(U, G, W, d, bf16, weight, Qw, ws.sigma, st), &n))) return s;
  const bool tc = !(flags & ROTATEK_SIMT_ONLY) && rk::cov_tc_supported(d, bf16);
  if ((s = launched(tc ? rk::launch_cov_tc(U, N, true, K, ws, st, /*allow_fused=*/false)
                       : rk::launch_cov(U, N, d, bf16, K, ws, st),
                    &n)))
    return s;
  if ((s = launched(rk::launch_state_accumulate(U, N, d, state_units, weight, ws, state, st), &n))) return s;
  g_launches = n;
  return ROTATEK_OK;
}

rotatek_status rotatek_calibrate_from_state(const rotatek_dims* dm, uint32_t flags, const double* state,
                                            float* R, float* dmu, float* eigvals, uint32_t* keep_mask,
                                            int32_t* keep_idx, float* R_full, int32_t* info, void* workspace,
                                            size_t workspace_bytes, rotatek_stream_t stream) {
  begin_call();
  rotatek_status s = check_dims(dm);
  if (s != ROTATEK_OK) return s;
  const int U = dm->units, d = dm->head_dim, r = dm->rank;
  const bool bf16 = dm->dtype == ROTATEK_BF16;
  const bool weight = (flags & ROTATEK_QUERY_WEIGHT) != 0;
  const bool center = (flags & ROTATEK_CENTER) != 0;
  const bool fp64 = !bf16 || (flags & ROTATEK_EIG_FP64);
  if (!state || !R || !dmu) return fail(ROTATEK_ERR_NULL, "state, R and dmu are required");
  if (d > 128) return fail(ROTATEK_ERR_UNSUPPORTED, "calibrate supports head_dim <= 128");
  const void* ptrs[] = {state, R, dmu, eigvals, keep_mask, keep_idx, R_full, info, workspace};
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  rk::CalibWs ws;
  const size_t need = rk::calib_ws_layout(U, d, 1, true, workspace, &ws);
  if (!workspace || workspace_bytes < need) return fail(ROTATEK_ERR_WORKSPACE, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int n = 0;
  if ((s = launched(rk::launch_state_finalize(U, d, center, weight, state, ws, st), &n))) return s;
  if ((s = launched(rk::launch_jacobi(U, d, r, fp64, (flags & ROTATEK_EIG_TWOSIDED) != 0, ws, st), &n))) return s;
  if ((s = launched(rk::launch_select_gather(U, d, r, /*fp64_vecs=*/true, bf16, center, ws, R, dmu, eigvals,
                                             keep_mask, keep_idx, R_full, info, st), &n)))
    return s;
  g_launches = n;
  return ROTATEK_OK;
}

namespace {
rotatek_status compress_impl(const rotatek_dims* dm, int32_t r_units, const void* K, const rk::TokSrc& tsrc,
                             const float* R, void* K_comp, uint32_t flags, rotatek_stream_t stream) {
  rotatek_status s = check_dims(dm);
  if (s != ROTATEK_OK) return s;
  if (!K || !R || !K_comp) return fail(ROTATEK_ERR_NULL, "K, R and K_comp are required");
  if (!aligned16(K) || !aligned16(R) || !aligned16(K_comp))
    return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  const int d = dm->head_dim, r = dm->rank;
  if (r_units < 0 || (r_units > 0 && dm->units % r_units != 0))
    return fail(ROTATEK_ERR_DIMS, "r_units must divide units (0: one rotation per unit)");
  const bool bf16 = dm->dtype == ROTATEK_BF16;
  const bool tc = !(flags & ROTATEK_SIMT_ONLY) && rk::compress_tc_supported(d, r, bf16);
  if (tsrc.active() && !tc)
    return fail(ROTATEK_ERR_UNSUPPORTED, "token lists / per-unit lengths need the tensor-core path (bf16, d = 128)");
  if (!tc && ((size_t)d * r + 64 * (size_t)d) * 4 > 227 * 1024)
    return fail(ROTATEK_ERR_UNSUPPORTED, "compress: d*r too large");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int n = 0;
  if ((s = launched(tc ? rk::launch_compress_tc(dm->units, dm->n_vis, r, K, R, K_comp, st, r_units, tsrc)
                       : rk::launch_compress(dm->units, dm->n_vis, d, r, bf16, K, R, K_comp, st, r_units),
                    &n)))
    return s;
  g_launches = n;
  return ROTATEK_OK;
}
}  // namespace

rotatek_status rotatek_compress_kv_ex2(const rotatek_dims* dm, int32_t r_units, const void* K, const float* R,
                                      void* K_comp, uint32_t flags, rotatek_stream_t stream) {
  begin_call();
  return compress_impl(dm, r_units, K, rk::TokSrc(), R, K_comp, flags, stream);
}

rotatek_status rotatek_compress_kv_tokens(const rotatek_dims* dm, int32_t r_units, const void* K, int32_t n_src,
                                         const int32_t* tok_idx, const int32_t* n_vis_u, const float* R,
                                         void* K_comp, rotatek_stream_t stream) {
  begin_call();
  if ((tok_idx && !aligned16(tok_idx)) || (n_vis_u && !aligned16(n_vis_u)))
    return fail(ROTATEK_ERR_ALIGN, "token arrays not 16-byte aligned");
  if (tok_idx && n_src < 1) return fail(ROTATEK_ERR_DIMS, "n_src must be >= 1 with a token list");
  rk::TokSrc tsrc;
  tsrc.idx = tok_idx;
  tsrc.nvu = n_vis_u;
  tsrc.n_src = tok_idx ? n_src : (dm ? dm->n_vis : 0);
  return compress_impl(dm, r_units, K, tsrc, R, K_comp, 0u, stream);
}

rotatek_status rotatek_compress_kv_ex(const rotatek_dims* dm, const void* K, const float* R,
                                      void* K_comp, uint32_t flags, rotatek_stream_t stream) {
  return rotatek_compress_kv_ex2(dm, 0, K, R, K_comp, flags, stream);
}

rotatek_status rotatek_compress_kv(const rotatek_dims* dm, const void* K, const float* R,
                                   void* K_comp, rotatek_stream_t stream) {
  return rotatek_compress_kv_ex(dm, K, R, K_comp, 0u, stream);
}

rotatek_status rotatek_decode_attn_varlen(const rotatek_dims* dm, int32_t r_units,
                                         const int32_t* n_vis_u, const int32_t* n_text_u,
                                         const void* q, const void* K_comp, const void* V,
                                         const float* R, const float* dmu, const void* K_text,
                                         const void* V_text, float softmax_scale, float* out,
                                         void* workspace, size_t workspace_bytes, int32_t splits,
                                         int32_t kernel, rotatek_stream_t stream) {
  begin_call();
  if ((n_vis_u && !aligned16(n_vis_u)) || (n_text_u && !aligned16(n_text_u)))
    return fail(ROTATEK_ERR_ALIGN, "length arrays not 16-byte aligned");
  rotatek_status s = check_dims(dm);
  if (s != ROTATEK_OK) return s;
  const int M = dm->n_text;
  if (!q || !K_comp || !V || !R || !out) return fail(ROTATEK_ERR_NULL, "q, K_comp, V, R, out are required");
  if (M > 0 && (!K_text || !V_text)) return fail(ROTATEK_ERR_NULL, "K_text/V_text required when n_text > 0");
  const void* ptrs[] = {q, K_comp, V, R, dmu, K_text, V_text, out, workspace};
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  rk::DecodeWs ws;
  const size_t need = rk::decode_ws_layout(dm->units, dm->group, dm->head_dim, dm->rank, dm->n_vis, M,
                                           workspace, &ws);
  if (!workspace || workspace_bytes < need) return fail(ROTATEK_ERR_WORKSPACE, "workspace too small");
  const int overlap = (kernel & ROTATEK_DECODE_OVERLAP) ? 1 : 0;
  kernel &= ~ROTATEK_DECODE_OVERLAP;
  if (kernel < 0 || kernel > 5) return fail(ROTATEK_ERR_DIMS, "kernel must be 0..5 (| ROTATEK_DECODE_OVERLAP)");
  if (r_units < 0 || (r_units > 0 && dm->units % r_units != 0))
    return fail(ROTATEK_ERR_DIMS, "r_units must divide units (0: one rotation per unit)");
  rk::DecodeArgs a;
  a.U = dm->units; a.G = dm->group; a.d = dm->head_dim; a.r = dm->rank; a.N = dm->n_vis; a.M = M;
  a.bf16 = dm->dtype == ROTATEK_BF16;
  a.q = q; a.Kc = K_comp; a.V = V; a.R = R; a.dmu = dmu;
  a.Kt = M > 0 ? K_text : nullptr; a.Vt = M > 0 ? V_text : nullptr;
  a.Ms = dm->text_stride > 0 ? dm->text_stride : M;
  a.scale = softmax_scale > 0.f ? softmax_scale : 1.0f / sqrtf((float)dm->head_dim);
  a.out = out;
  a.nR = r_units;
  a.overlap = overlap;
  a.nvu = n_vis_u;
  a.ntu = dm->n_text > 0 ? n_text_u : nullptr;
  int n = 0;
  if ((s = launched(rk::launch_decode(a, ws, splits, kernel, reinterpret_cast<cudaStream_t>(stream)), &n)))
    return s;
  g_launches = n;
  return ROTATEK_OK;
}

rotatek_status rotatek_decode_attn_ex2(const rotatek_dims* dm, int32_t r_units, const void* q, const void* K_comp,
                                      const void* V, const float* R, const float* dmu,
                                      const void* K_text, const void* V_text, float softmax_scale,
                                      float* out, void* workspace, size_t workspace_bytes,
                                      int32_t splits, int32_t kernel, rotatek_stream_t stream) {
  return rotatek_decode_attn_varlen(dm, r_units, nullptr, nullptr, q, K_comp, V, R, dmu, K_text,
                                    V_text, softmax_scale, out, workspace, workspace_bytes, splits,
                                    kernel, stream);
}

rotatek_status rotatek_decode_attn_ex(const rotatek_dims* dm, const void* q, const void* K_comp,
                                      const void* V, const float* R, const float* dmu,
                                      const void* K_text, const void* V_text, float softmax_scale,
                                      float* out, void* workspace, size_t workspace_bytes,
                                      int32_t splits, int32_t kernel, rotatek_stream_t stream) {
  return rotatek_decode_attn_ex2(dm, 0, q, K_comp, V, R, dmu, K_text, V_text, softmax_scale, out, workspace,
                                 workspace_bytes, splits, kernel, stream);
}

rotatek_status rotatek_decode_attn(const rotatek_dims* dm, const void* q, const void* K_comp,
                                   const void* V, const float* R, const float* dmu,
                                   const void* K_text, const void* V_text, float softmax_scale,
                                   float* out, void* workspace, size_t workspace_bytes,
                                   rotatek_stream_t stream) {
  return rotatek_decode_attn_ex(dm, q, K_comp, V, R, dmu, K_text, V_text, softmax_scale, out,
                                workspace, workspace_bytes, 0, 0, stream);
}

rotatek_status rotatek_decode_attn_partial(const rotatek_dims* dm, const void* q, const void* K_comp,
                                           const void* V, const float* R, const float* dmu,
                                           const void* K_text, const void* V_text, float softmax_scale,
                                           float* part, void* workspace, size_t workspace_bytes,
                                           rotatek_stream_t stream) {
  begin_call();
  rotatek_status s = check_dims(dm);
  if (s != ROTATEK_OK) return s;
  const int M = dm->n_text;
  if (!q || !K_comp || !V || !R || !part) return fail(ROTATEK_ERR_NULL, "q, K_comp, V, R, part are required");
  if (M > 0 && (!K_text || !V_text)) return fail(ROTATEK_ERR_NULL, "K_text/V_text required when n_text > 0");
  const void* ptrs[] = {q, K_comp, V, R, dmu, K_text, V_text, workspace};
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(part) & 3u) return fail(ROTATEK_ERR_ALIGN, "part not 4-byte aligned");
  rk::DecodeWs ws;
  const size_t need = rk::decode_ws_layout(dm->units, dm->group, dm->head_dim, dm->rank, dm->n_vis, M,
                                           workspace, &ws);
  if (!workspace || workspace_bytes < need) return fail(ROTATEK_ERR_WORKSPACE, "workspace too small");
  rk::DecodeArgs a;
  a.U = dm->units; a.G = dm->group; a.d = dm->head_dim; a.r = dm->rank; a.N = dm->n_vis; a.M = M;
  a.bf16 = dm->dtype == ROTATEK_BF16;
  a.q = q; a.Kc = K_comp; a.V = V; a.R = R; a.dmu = dmu;
  a.Kt = M > 0 ? K_text : nullptr; a.Vt = M > 0 ? V_text : nullptr;
  a.Ms = dm->text_stride > 0 ? dm->text_stride : M;
  a.scale = softmax_scale > 0.f ? softmax_scale : 1.0f / sqrtf((float)dm->head_dim);
  a.out = nullptr;
  a.pout = part;
  int n = 0;
  if ((s = launched(rk::launch_decode(a, ws, 0, 0, reinterpret_cast<cudaStream_t>(stream)), &n))) return s;
  g_launches = n;
  return ROTATEK_OK;
}

rotatek_status rotatek_gather_tokens(int32_t units, int32_t n_src, int32_t n_keep, int32_t row_bytes,
                                     const int32_t* keep_idx, const void* src, void* dst, int32_t* err,
                                     rotatek_stream_t stream) {
  begin_call();
  if (units < 1 || n_src < 1 || n_keep < 1 || row_bytes < 16 || row_bytes % 16 != 0)
    return fail(ROTATEK_ERR_DIMS, "bad gather dims (row_bytes: positive multiple of 16)");
  if (!keep_idx || !src || !dst) return fail(ROTATEK_ERR_NULL, "keep_idx, src and dst are required");
  if (!aligned16(src) || !aligned16(dst) || (reinterpret_cast<uintptr_t>(keep_idx) & 3u))
    return fail(ROTATEK_ERR_ALIGN, "src/dst 16-byte, keep_idx 4-byte alignment");
  int n = 0;
  rotatek_status s = launched(rk::launch_gather_rows(units, n_src, n_keep, row_bytes, keep_idx, src, dst, err,
                                                     reinterpret_cast<cudaStream_t>(stream)), &n);
  if (s) return s;
  g_launches = n;
  return ROTATEK_OK;
}

rotatek_status rotatek_merge_partials(int32_t units, int32_t group, int32_t head_dim, int32_t nparts,
                                      const float* parts, float* out, rotatek_stream_t stream) {
  begin_call();
  if (units < 1 || group < 1 || head_dim < 1 || head_dim > 256 || nparts < 1)
    return fail(ROTATEK_ERR_DIMS, "bad merge dims");
  if (!parts || !out) return fail(ROTATEK_ERR_NULL, "parts and out are required");
  if ((reinterpret_cast<uintptr_t>(parts) & 3u) || !aligned16(out))
    return fail(ROTATEK_ERR_ALIGN, "parts 4-byte / out 16-byte alignment");
  int n = 0;
  rotatek_status s = launched(rk::launch_merge_parts(units, group, head_dim, nparts, parts, out,
                                                     reinterpret_cast<cudaStream_t>(stream)), &n);
  if (s) return s;
  g_launches = n;
  return ROTATEK_OK;
}

rotatek_status rotatek_select_topr(int32_t units, int32_t head_dim, int32_t rank,
                                   const float* eigvals, uint32_t* keep_mask, int32_t* keep_idx,
                                   int32_t* info, rotatek_stream_t stream) {
  begin_call();
  if (units < 1 || head_dim < 1 || head_dim > 256 || rank < 1 || rank > head_dim)
    return fail(ROTATEK_ERR_DIMS, "bad select dims");
  if (!eigvals || !keep_mask || !keep_idx) return fail(ROTATEK_ERR_NULL, "eigvals, keep_mask, keep_idx required");
  if (!aligned16(eigvals) || !aligned16(keep_mask) || !aligned16(keep_idx) || (info && !aligned16(info)))
    return fail(ROTATEK_ERR_ALIGN, "pointer not 16-byte aligned");
  int n = 0;
  rotatek_status s = launched(rk::launch_select_only(units, head_dim, rank, eigvals, keep_mask,
                                                     keep_idx, info, reinterpret_cast<cudaStream_t>(stream)), &n);
  if (s) return s;
  g_launches = n;
  return ROTATEK_OK;
}

}  // extern "C"
