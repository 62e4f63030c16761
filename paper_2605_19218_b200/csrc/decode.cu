// decode.cu -- Alg. 2 (alg:rotatek-decode) on sm_100a.
//
// For every unit u (= batch x KV head) and query head g of the unit:
//   q~ = q R_r ; b = q . dmu                                  (Alg. 2 l.1-2; App. C)
//   s_vis[n] = (q~ . K~[n] + b) / sqrt(d)   s_pt[m] = q . K_t[m] / sqrt(d)   (l.3-4)
//   out = softmax([s_vis; s_pt]) [V; V_t]                      (l.5-6)
// computed with an exact online-softmax split over the token axis (App. C "standard
// online-softmax merge").  Scores are kept in log2 units: q~, b and q are
// pre-multiplied by scale*log2(e) so every exponential is one ex2.approx.
//
// Two implementations behind one launcher:
//  * decode_fast_kernel (d = 128; r in {16, 32, 64, 128}; G in {1, 7}): a persistent,
//    perfectly balanced streaming kernel.  The U*(N+M) tokens of the whole batch are
//    cut into one contiguous range per WARP; each warp streams its range through its
//    own ring of shared-memory stages filled by 1-D TMA bulk copies
//    (cp.async.bulk + mbarrier complete_tx, SASS UBLKCP), K~ tile then V tile, so every
//    byte of the compacted cache is read exactly once with no CTA-level barriers.  The
//    query rotation (q~ = q R_r, b = q . dmu) is fused: the warp that starts a unit
//    rotates that unit's queries itself (rotate_query), so a decode is ONE launch.  At
//    every unit boundary the warp flushes an online-softmax partial (m, l, acc[G][d]);
//    the last warp to finish a unit (atomic ticket) merges that unit's partials in slot
//    order (deterministic) and writes out, then re-arms the ticket (graph-replay safe).
//  * decode_generic_kernel (any d <= 256, any r, any G): one CTA per (unit, split),
//    plain loads, per-token online softmax.  Used for the toy shapes and fallbacks.
#include <cstdio>
#include <cstdlib>

#include <cstring>
#include <type_traits>

#include "decode_common.cuh"

namespace rk {

// diagnostics stamp k of warp gw (lane 0 only; no-op unless a trace buffer is installed)
#define RK_TRACE(k, v)                                                              \
  do {                                                                              \
    if (p.trace != nullptr && lane == 0 && w < p.aw) p.trace[(size_t)gw * 8 + (k)] = (v); \
  } while (0)

// diagnostics hook of the CALLING THREAD (rotatek_debug_decode_trace); null unless a test or
// tool installed a buffer, so ordinary calls share no state
static thread_local unsigned long long* g_trace = nullptr;

// max units one CTA's token range can touch (its query table must hold them all)
static int cta_units_max(int U, int N, int M, int NW, int warps) {
  const long long L = (long long)N + M, T = L * U;
  const long long per = (T + NW - 1) / NW + 1;  // >= any warp's range length
  long long n = (per * warps + L - 2) / L + 1;
  return n > U ? U : (int)n;
}
// streaming warps per CTA such that one CTA's units fit its query table (tiny units only
// lower it below WARPS); 0 if even one warp's range touches more than cap units
static int active_warps(int U, int N, int M, int NW, int warps, int cap) {
  for (int aw = warps; aw >= 1; --aw)
    if (cta_units_max(U, N, M, NW, aw) <= cap) return aw;
  return 0;
}

// =====================================================================================
// generic kernel
// =====================================================================================
constexpr int kGenWarps = 4;

template <typename T>
__global__ void __launch_bounds__(kGenWarps * 32) decode_generic_kernel(DecodeParams p, int splits) {
  extern __shared__ __align__(16) float gsm[];
  const int G = p.G, d = p.d, r = p.r;
  float* qs = gsm;                    // [G][d]   scaled q
  float* qt = qs + G * d;             // [G][r]   scaled q~
  float* bias = qt + G * r;           // [G]
  float* wm = bias + G;               // [W][G]
  float* wl = wm + kGenWarps * G;     // [W][G]
  float* wacc = wl + kGenWarps * G;   // [W][G][d]
  __shared__ int s_last;

  const int split = blockIdx.x, u = blockIdx.y;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const T* q = static_cast<const T*>(p.q) + (size_t)u * G * d;
  for (int e = tid; e < G * d; e += blockDim.x) qs[e] = Elem<T>::to_f(q[e]);
  __syncthreads();
  const float* Ru = p.R + (size_t)(u % p.nR) * d * r;
  for (int e = tid; e < G * r; e += blockDim.x) {
    const int g = e / r, k = e % r;
    float s = 0.f;
    for (int i = 0; i < d; ++i) s = fmaf(qs[g * d + i], Ru[(size_t)i * r + k], s);
    qt[e] = s * p.sl;
  }
  for (int g = w; g < G; g += kGenWarps) {
    float s = 0.f;
    if (p.dmu)
      for (int i = lane; i < d; i += 32) s = fmaf(qs[g * d + i], p.dmu[(size_t)(u % p.nR) * d + i], s);
    s = warp_sum(s);
    if (lane == 0) bias[g] = s * p.sl;
  }
  for (int e = tid; e < kGenWarps * G; e += blockDim.x) { wm[e] = -CUDART_INF_F; wl[e] = 0.f; }
  for (int e = tid; e < kGenWarps * G * d; e += blockDim.x) wacc[e] = 0.f;
  __syncthreads();
  for (int e = tid; e < G * d; e += blockDim.x) qs[e] *= p.sl;
  __syncthreads();

  const int n0 = (int)((long long)p.N * split / splits), n1 = (int)((long long)p.N * (split + 1) / splits);
  const int m0 = (int)((long long)p.M * split / splits), m1 = (int)((long long)p.M * (split + 1) / splits);
  const int total = (n1 - n0) + (m1 - m0);
  const int nv_u = p.nvu ? __ldg(p.nvu + u) : p.N, nt_u = p.ntu ? __ldg(p.ntu + u) : p.M;
  for (int idx = w; idx < total; idx += kGenWarps) {
    const bool vis = idx < n1 - n0;
    if (vis ? (n0 + idx >= nv_u) : (m0 + idx - (n1 - n0) >= nt_u)) continue;  // padding
    const T* krow;
    const T* vrow;
    int kw;
    if (vis) {
      const int t = n0 + idx;
      krow = static_cast<const T*>(p.Kc) + ((size_t)u * p.N + t) * r;
      vrow = static_cast<const T*>(p.V) + ((size_t)u * p.N + t) * d;
      kw = r;
    } else {
      const int t = m0 + idx - (n1 - n0);
      krow = static_cast<const T*>(p.Kt) + ((size_t)u * p.Ms + t) * d;
      vrow = static_cast<const T*>(p.Vt) + ((size_t)u * p.Ms + t) * d;
      kw = d;
    }
    for (int g = 0; g < G; ++g) {
      float s = 0.f;
      const float* qq = vis ? qt + g * r : qs + g * d;
      for (int c = lane; c < kw; c += 32) s = fmaf(qq[c], Elem<T>::to_f(krow[c]), s);
      s = warp_sum(s);
      if (vis) s += bias[g];
      const float m_old = wm[w * G + g];
      const float m_new = fmaxf(m_old, s);
      const float alpha = fast_exp2(m_old - m_new);
      const float pr = fast_exp2(s - m_new);
      float* acc = wacc + (size_t)(w * G + g) * d;
      for (int c = lane; c < d; c += 32) acc[c] = fmaf(acc[c], alpha, pr * Elem<T>::to_f(vrow[c]));
      const float l_new = wl[w * G + g] * alpha + pr;
      __syncwarp();
      if (lane == 0) { wm[w * G + g] = m_new; wl[w * G + g] = l_new; }
      __syncwarp();
    }
  }
  __syncthreads();
  // CTA merge of the warps, then either final output or a split partial
  float* part = p.partials;
  for (int e = tid; e < G * d; e += blockDim.x) {
    const int g = e / d, c = e % d;
    float M = -CUDART_INF_F;
    for (int ww = 0; ww < kGenWarps; ++ww) M = fmaxf(M, wm[ww * G + g]);
    float L = 0.f, A = 0.f;
    for (int ww = 0; ww < kGenWarps; ++ww) {
      const float mw = wm[ww * G + g];
      const float f = (mw == -CUDART_INF_F) ? 0.f : fast_exp2(mw - M);
      L = fmaf(wl[ww * G + g], f, L);
      A = fmaf(wacc[(size_t)(ww * G + g) * d + c], f, A);
    }
    if (splits == 1) {
      if (p.pout) {
        float* po = p.pout + ((size_t)u * G + g) * (d + 2);
        po[c] = A;
        if (c == 0) { po[d] = M; po[d + 1] = L; }
      } else {
        p.out[((size_t)u * G + g) * d + c] = A / L;
      }
    } else {
      float* dst = part + (((size_t)u * G + g) * splits + split) * (d + 2);
      if (c == 0) { dst[0] = M; dst[1] = L; }
      dst[2 + c] = A;
    }
  }
  if (splits == 1) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.counters[u], 1u) == (unsigned)(splits - 1));
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = tid; e < G * d; e += blockDim.x) {
    const int g = e / d, c = e % d;
    const float* src = part + ((size_t)u * G + g) * splits * (d + 2);
    float M = -CUDART_INF_F;
    for (int s = 0; s < splits; ++s) M = fmaxf(M, __ldcg(src + (size_t)s * (d + 2)));
    float L = 0.f, A = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float ms = __ldcg(src + (size_t)s * (d + 2));
      const float f = (ms == -CUDART_INF_F) ? 0.f : fast_exp2(ms - M);
      L = fmaf(__ldcg(src + (size_t)s * (d + 2) + 1), f, L);
      A = fmaf(__ldcg(src + (size_t)s * (d + 2) + 2 + c), f, A);
    }
    if (p.pout) {
      float* po = p.pout + ((size_t)u * G + g) * (d + 2);
      po[c] = A;
      if (c == 0) { po[d] = M; po[d + 1] = L; }
    } else {
      p.out[((size_t)u * G + g) * d + c] = A / L;
    }
  }
  if (tid == 0) p.counters[u] = 0u;
}

#include "decode_fast.cuh"
#include "decode_gqa.cuh"
#include "decode_steal.cuh"

// =====================================================================================
// host side
// =====================================================================================
struct FastPlan {
  int NW;     // active warps
  int cmax;   // max contributing warps per unit
};

constexpr int kMaxWarpsPerSM = 16;  // bound used to size the partial workspace

static int num_sms() {
  static int slot[kMaxDevices];
  return once_per_device(slot, [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = kNumSMs;
    return v;
  });
}

static FastPlan fast_plan(int U, int N, int M, int warps_per_sm, int min_tokens = 64) {
  FastPlan pl;
  const long long T = (long long)U * (N + M);
  long long nw = (long long)num_sms() * warps_per_sm;
  const long long by_size = T / min_tokens > 0 ? T / min_tokens : 1;  // >= min_tokens per warp
  if (by_size < nw) nw = by_size;
  // at most 126 warps per unit, so a unit's partials (<= 128) fit the merge scratch
  if (nw > 126LL * U) nw = 126LL * U;
  if (nw < 1) nw = 1;
  pl.NW = (int)nw;
  // a unit spans at most ceil(L / min_range) + 1 warps; min_range >= floor(T/NW)
  const long long L = (long long)N + M;
  const long long minr = T / pl.NW;
  pl.cmax = (int)((L + minr - 1) / (minr > 0 ? minr : 1)) + 2;
  return pl;
}

int decode_max_splits(int U, int N, int M) {
  int s = (4 * kNumSMs + U - 1) / U;
  int cap = (N + M + 63) / 64;
  if (s > cap) s = cap;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  return s;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// partial slots per unit under work stealing: the static contributors, plus one per stolen
// piece overlapping the unit -- pieces are disjoint and >= smin tokens long, so all but two
// of them lie inside the unit
static int steal_cmax(int static_cmax, int N, int M, int smin) {
  return static_cmax + (N + M + smin - 1) / smin + 3;
}
constexpr int kStealMin = 64;  // smallest claim / steal granule any configuration uses

size_t decode_ws_layout(int U, int G, int d, int r, int N, int M, void* base, DecodeWs* ws) {
  const FastPlan pl = fast_plan(U, N, M, kMaxWarpsPerSM);  // worst case: most warps per unit
  const int smax = 64;  // explicit splits (rotatek_decode_attn_ex) may ask for up to 64
  size_t gen = (size_t)U * G * smax * (d + 2) * 4;
  size_t fast = (size_t)U * steal_cmax(pl.cmax, N, M, kStealMin) * G * (d + 4) * 4;
  size_t part = gen > fast ? gen : fast;
  // the regions that must be zero (or exhausted) on entry come first and their offsets
  // depend on U only, so a caller may reuse one zero-filled buffer (grown when needed) for
  // every shape with the same U; the scratch partials (no initial state) come last
  char* b = static_cast<char*>(base);
  size_t off = 0;
  DecodeWs w;
  w.counters = (uint32_t*)(b ? b + off : nullptr);
  off += al256((size_t)U * 4);
  w.nslot = (uint32_t*)(b ? b + off : nullptr);
  off += al256((size_t)U * 4);
  w.desc = (unsigned long long*)(b ? b + off : nullptr);
  off += al256((size_t)kMaxStealWarps * 8);
  w.partials = (float*)(b ? b + off : nullptr);
  off += al256(part);
  w.partial_bytes = part;
  w.max_splits = smax;
  if (ws) *ws = w;
  return off;
}

template <typename T, int RK, int G, int WARPS, int STAGES, int TTV, int MINB>
static int launch_fast_cfg(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  using C = FastCfg<T, RK, G, WARPS, STAGES, TTV>;
  static_assert(C::SMEM <= 227 * 1024, "shared memory");
  auto kern = decode_fast_kernel<T, RK, G, WARPS, STAGES, TTV, MINB>;
  static int cps_slot[kMaxDevices];
  const int ctas_per_sm = once_per_device(cps_slot, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, WARPS * 32, C::SMEM) != cudaSuccess || n < 1)
      n = 1;
    if (n * WARPS > kMaxWarpsPerSM) n = kMaxWarpsPerSM / WARPS;
    return n < 1 ? 1 : n;
  });
  const FastPlan pl = fast_plan(a.U, a.N, a.M, ctas_per_sm * WARPS);
  const int aw = active_warps(a.U, a.N, a.M, pl.NW, WARPS, C::CAP);
  if (aw < 1) return -3;  // the CTA query table cannot hold one warp's units
  const int ctas = (pl.NW + aw - 1) / aw;
  DecodeParams p{a.U, a.G, a.d, a.r, a.N, a.M, a.q, a.Kc, a.V, a.R, a.dmu, a.Kt, a.Vt,
                 a.scale * kLog2e, a.out, ws.counters, ws.partials, g_trace, aw, a.pout, a.nR > 0 ? a.nR : a.U,
                 nullptr, nullptr, a.overlap, a.Ms, a.nvu, a.ntu};
  if (!(a.overlap ? launch_overlap(kern, ctas, WARPS * 32, C::SMEM, st, p, pl.NW, pl.cmax)
                  : launch(kern, ctas, WARPS * 32, C::SMEM, st, p, pl.NW, pl.cmax)))
    return -1;
  return 1;
}

// work-stealing variant of launch_fast_cfg (decode_steal.cuh)
template <typename T, int RK, int G, int WARPS, int STAGES, int TTV, int MINB>
static int launch_steal_cfg(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  using C = StealCfg<T, RK, G, WARPS, STAGES, TTV>;
  static_assert(C::SMEM <= 227 * 1024, "shared memory");
  auto kern = decode_steal_kernel<T, RK, G, WARPS, STAGES, TTV, MINB>;
  static int cps_slot[kMaxDevices];
  const int ctas_per_sm = once_per_device(cps_slot, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, WARPS * 32, C::SMEM) != cudaSuccess || n < 1)
      n = 1;
    if (n * WARPS > kMaxWarpsPerSM) n = kMaxWarpsPerSM / WARPS;
    return n < 1 ? 1 : n;
  });
  const FastPlan pl = fast_plan(a.U, a.N, a.M, ctas_per_sm * WARPS);
  if (pl.NW > kMaxStealWarps || (long long)a.U * (a.N + a.M) >= (1LL << 31)) return -3;
  const int aw = active_warps(a.U, a.N, a.M, pl.NW, WARPS, C::CAP);
  if (aw < 1) return -3;
  const int ctas = (pl.NW + aw - 1) / aw;
  const int claim = 2 * TTV;  // == smin (>= kStealMin): thief runs are >= one claim long
  const int cmax = steal_cmax(pl.cmax, a.N, a.M, claim);
  DecodeParams p{a.U, a.G, a.d, a.r, a.N, a.M, a.q, a.Kc, a.V, a.R, a.dmu, a.Kt, a.Vt,
                 a.scale * kLog2e, a.out, ws.counters, ws.partials, g_trace, aw, a.pout,
                 a.nR > 0 ? a.nR : a.U, ws.desc, ws.nslot, 0, a.Ms, a.nvu, a.ntu};
  if (!launch(kern, ctas, WARPS * 32, C::SMEM, st, p, pl.NW, cmax, claim, claim)) return -1;
  return 1;
}


// Default configuration per shape: 16 resident warps per SM (2 CTAs x 8 warps), one
// 32-token (bf16) stage per warp -- the tuning sweep (profiles/) showed per-SM warp count
// matters more than per-warp ring depth.  Larger rows (r = 128, fp32) shrink TTV so that
// the per-warp ring still fits two CTAs per SM.
template <typename T, int RK, int G>
static int launch_fast_default(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  constexpr int TTV = (sizeof(T) == 2) ? (RK >= 128 ? 16 : 32) : 16;
  if constexpr (G == 1) {
    // 8 warps x one 64-token stage (LLaVA b32: 96% of the measured copy bandwidth in the
    // sweep of profiles/decode_tuning_r1.md); fall back to 32/16-token tiles if the ring
    // does not fit.
    constexpr int T64 = FastCfg<T, RK, G, 8, 1, 64>::SMEM <= 227 * 1024 ? 64
                      : FastCfg<T, RK, G, 8, 1, 32>::SMEM <= 227 * 1024 ? 32 : 16;
    return launch_fast_cfg<T, RK, G, 8, 1, T64, 1>(a, ws, st);
  } else {
    // GQA on CUDA cores: register-heavy (G accumulator sets), one CTA of <= 8 warps per SM
    constexpr int STG = FastCfg<T, RK, G, 8, 2, TTV>::SMEM <= 227 * 1024 ? 2 : 1;
    constexpr int PER = FastCfg<T, RK, G, 1, STG, TTV>::SMEM;
    constexpr int W = (227 * 1024) / PER < 8 ? (227 * 1024) / PER : 8;
    return launch_fast_cfg<T, RK, G, W, STG, TTV, 1>(a, ws, st);
  }
}

// tuning variants (ROTATEK_DECODE_CFG="warps,stages,tile") for the headline shapes
template <typename T, int G>
static int launch_fast_r32(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  static int cfg = [] {
    const char* e = getenv("ROTATEK_DECODE_CFG");
    int w = 0, s = 0, t = 0;
    if (e && sscanf(e, "%d,%d,%d", &w, &s, &t) == 3) return w * 1000 + s * 100 + t;
    return 0;
  }();
  if constexpr (sizeof(T) == 2 && G == 1) switch (cfg) {
    case 8132: return launch_fast_cfg<T, 32, G, 8, 1, 32, 2>(a, ws, st);
    case 8232: return launch_fast_cfg<T, 32, G, 8, 2, 32, 1>(a, ws, st);
    case 16132: return launch_fast_cfg<T, 32, G, 16, 1, 32, 1>(a, ws, st);
    case 4264: return launch_fast_cfg<T, 32, G, 4, 2, 64, 1>(a, ws, st);
    case 41128: return launch_fast_cfg<T, 32, G, 4, 1, 128, 1>(a, ws, st);
    case 10148: return launch_fast_cfg<T, 32, G, 10, 1, 48, 1>(a, ws, st);
    default: break;
  }
  // short units (joint token+channel pruning, N+M <= 2048): two 32-token stages per warp
  // keep a tile in flight across the frequent unit-boundary flushes (joint_b64: 117 vs
  // 128 us/layer in the tools/time_decode.py sweep); long units keep one 64-token stage
  if constexpr (sizeof(T) == 2 && G == 1) {
    if (a.N + a.M <= 2048) return launch_fast_cfg<T, 32, G, 8, 2, 32, 1>(a, ws, st);
  }
  return launch_fast_default<T, 32, G>(a, ws, st);
}

template <typename T>
static int launch_fast_rk(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  if (a.G == 1) {
    switch (a.r) {
      case 16: return launch_fast_default<T, 16, 1>(a, ws, st);
      case 32: return launch_fast_r32<T, 1>(a, ws, st);
      case 64: return launch_fast_default<T, 64, 1>(a, ws, st);
      case 128: return launch_fast_default<T, 128, 1>(a, ws, st);
    }
  } else if (a.G == 7) {
    switch (a.r) {
      case 16: return launch_fast_default<T, 16, 7>(a, ws, st);
      case 32: return launch_fast_r32<T, 7>(a, ws, st);
      case 64: return launch_fast_default<T, 64, 7>(a, ws, st);
      case 128: return launch_fast_default<T, 128, 7>(a, ws, st);
    }
  }
  return -2;
}

static bool fast_supported(const DecodeArgs& a) {
  if (a.d != kD) return false;
  if (!(a.r == 16 || a.r == 32 || a.r == 64 || a.r == 128)) return false;
  if (!(a.G == 1 || a.G == 7)) return false;
  if (a.M > 0 && (a.Kt == nullptr || a.Vt == nullptr)) return false;
  return true;
}

// ------------------------------------------------------------- tensor-core GQA launcher
template <int RK, int G, int TTV, int STAGES, int MAXW, bool STEAL>
constexpr int gqa_warps() {
  using C1 = GqaCfg<RK, G, 1, TTV, STAGES, STEAL>;
  constexpr int per = C1::WARP_SMEM + (STEAL ? C1::ENT : 0);
  constexpr int w = (227 * 1024 - 1024 - C1::CAP * C1::ENT) / per;
  return w > MAXW ? MAXW : w;
}

template <int RK, int G, int TTV, int STAGES, bool STEAL, int MAXW = 8>
static int launch_gqa_cfg(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  constexpr int WARPS = gqa_warps<RK, G, TTV, STAGES, MAXW, STEAL>();
  using C = GqaCfg<RK, G, WARPS, TTV, STAGES, STEAL>;
  static_assert(C::SMEM <= 227 * 1024, "shared memory");
  if ((long long)a.U * (a.N + a.M) >= (1LL << 31)) return -3;  // 32-bit token positions
  GqaMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (!encode_tmap_3d_bf16(&maps.kc, a.Kc, RK, a.N, a.U, RK, C::TT, RK * 2)) return -2;
  if (!encode_tmap_3d_bf16(&maps.v, a.V, kD, a.N, a.U, 64, C::TT, 128)) return -2;
  if (a.M > 0) {
    if (!encode_tmap_3d_bf16_strided(&maps.kt, a.Kt, kD, a.M, a.U, a.Ms, 64, C::TX, 128)) return -2;
    if (!encode_tmap_3d_bf16_strided(&maps.vt, a.Vt, kD, a.M, a.U, a.Ms, 64, C::TX, 128)) return -2;
  }
  auto kern = decode_gqa_kernel<RK, G, WARPS, TTV, STAGES, STEAL>;
  static int attr_slot[kMaxDevices];
  once_per_device(attr_slot, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    return 1;
  });
  // >= 96 tokens per warp (fewer, longer ranges on small shapes: Qwen b1 26 -> 23 us)
  const FastPlan pl = fast_plan(a.U, a.N, a.M, WARPS, 96);
  if (STEAL && pl.NW > kMaxStealWarps) return -3;
  const int aw = active_warps(a.U, a.N, a.M, pl.NW, WARPS, C::CAP);
  if (aw < 1) return -3;  // the CTA query table cannot hold one warp's units
  const int ctas = (pl.NW + aw - 1) / aw;
  const int claim = 2 * C::TT;
  const int cmax = STEAL ? steal_cmax(pl.cmax, a.N, a.M, claim) : pl.cmax;
  DecodeParams p{a.U, a.G, a.d, a.r, a.N, a.M, a.q, a.Kc, a.V, a.R, a.dmu, a.Kt, a.Vt,
                 a.scale * kLog2e, a.out, ws.counters, ws.partials, g_trace, aw, a.pout,
                 a.nR > 0 ? a.nR : a.U, ws.desc, ws.nslot, a.overlap, a.Ms, a.nvu, a.ntu};
  if (!(a.overlap ? launch_overlap(kern, ctas, WARPS * 32, C::SMEM, st, maps, p, pl.NW, cmax, claim)
                  : launch(kern, ctas, WARPS * 32, C::SMEM, st, maps, p, pl.NW, cmax, claim)))
    return -1;
  return 1;
}

// ring configuration (ROTATEK_GQA_CFG="tile,stages" for tuning; default one 64-token stage
// per warp, 8 warps per SM -- the sweep in profiles/ found deeper rings with smaller tiles
// no faster: the remaining gap on small-U shapes is fixed per-launch latency, not bytes
// in flight)
template <int RK, int G>
static int launch_gqa_t(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  static int cfg = [] {
    const char* e = getenv("ROTATEK_GQA_CFG");
    int t = 0, s = 0;
    if (e && sscanf(e, "%d,%d", &t, &s) == 2) return t * 10 + s;
    return 0;
  }();
  switch (cfg) {
    case 322: return launch_gqa_cfg<RK, G, 32, 2, false>(a, ws, st);
    case 641: return launch_gqa_cfg<RK, G, 64, 1, false>(a, ws, st);
    case 642: return launch_gqa_cfg<RK, G, 64, 2, false>(a, ws, st);
    default: break;
  }
  // r = 32, >= 64 units of <= 16K tokens: two 64-token stages per warp (fewer warps, so fewer
  // partials per unit, and each warp's next tile in flight during its compute): qwen b32
  // 44.8 -> 43.6 us, U = 64 x 4K tokens 37.3 -> 31.8; long units (32K), few units (U = 32:
  // 26.9 -> 28.9) and r = 64 keep one stage per warp and more warps (tools/time_decode.py)
  if (RK == 32 && a.U >= 64 && a.N + a.M <= 16384) return launch_gqa_cfg<RK, G, 64, 2, false>(a, ws, st);
  return launch_gqa_cfg<RK, G, 64, 1, false>(a, ws, st);
}

template <int RK>
static int launch_gqa_rk(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  switch (a.G) {
    case 2: return launch_gqa_t<RK, 2>(a, ws, st);
    case 4: return launch_gqa_t<RK, 4>(a, ws, st);
    case 7: return launch_gqa_t<RK, 7>(a, ws, st);
    case 8: return launch_gqa_t<RK, 8>(a, ws, st);
  }
  return -2;
}

static bool gqa_supported(const DecodeArgs& a) {
  return a.bf16 && a.d == kD && (a.r == 32 || a.r == 64) &&
         (a.G == 2 || a.G == 4 || a.G == 7 || a.G == 8) && (a.M == 0 || (a.Kt && a.Vt));
}

// kernel 4: the streaming kernels with work stealing (decode_steal.cuh).  Not the default:
// measured no faster on every bench shape (the stream phase already runs at the achievable
// HBM read rate; the per-warp finish spread is bandwidth sharing, and stealing adds claims,
// partial runs and rotations of stolen units).  Kept selectable, and tested.
static int launch_steal(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  if (!a.bf16 || a.d != kD || a.r != 32 || (a.M > 0 && (!a.Kt || !a.Vt))) return -2;
  if (a.G == 1) {
    if (a.N + a.M <= 2048) return launch_steal_cfg<__nv_bfloat16, 32, 1, 8, 2, 32, 1>(a, ws, st);
    return launch_steal_cfg<__nv_bfloat16, 32, 1, 8, 1, 64, 1>(a, ws, st);
  }
  if (a.G == 7) return launch_gqa_cfg<32, 7, 64, 1, true>(a, ws, st);
  return -2;
}

int launch_decode(const DecodeArgs& a, const DecodeWs& ws, int splits, int kernel, cudaStream_t st) {
  if (kernel == 4) {
    const int rc = launch_steal(a, ws, st);
    return rc == -3 ? -2 : rc;
  }
  const bool fast_ok = fast_supported(a);
  const bool gqa_ok = gqa_supported(a);
  const bool ring1_ok = a.bf16 && a.d == kD && (a.r == 32 || a.r == 64) && a.G == 1 && (a.M == 0 || (a.Kt && a.Vt));
  if ((kernel == 2 && !fast_ok) || (kernel == 3 && !gqa_ok && !ring1_ok) || (kernel == 5 && !gqa_ok)) return -2;
  // -3: the streaming kernels' CTA query table cannot hold the units of one CTA range
  // (tiny units, e.g. N + M < ~100 tokens); the generic kernel handles those shapes
  // G = 1: the CTA-ring kernel for small batches (<= 2 units per SM: one CTA per unit or unit
  // piece, DSMEM merges), the per-warp CUDA-core kernel for large ones (LLaVA b32: 1.02 of the
  // copy peak; the ring's query table holds <= 4 units per CTA)
  const bool ring1_auto = ring1_ok && a.U <= 2 * decode_num_sms();
  if (kernel == 3 || (kernel == 0 && (gqa_ok || ring1_auto) && splits <= 0)) {
    const int rc = launch_ring(a, ws, st);
    if (rc != -3) return rc;
    if (kernel == 3) return -2;
  } else if (kernel == 5) {  // the per-warp GQA kernel of round 1 (decode_gqa.cuh), for A/B
    const int rc = a.r == 32 ? launch_gqa_rk<32>(a, ws, st) : launch_gqa_rk<64>(a, ws, st);
    return rc == -3 ? -2 : rc;
  } else if ((kernel == 0 && fast_ok && splits <= 0) || kernel == 2) {
    const int rc = a.bf16 ? launch_fast_rk<__nv_bfloat16>(a, ws, st) : launch_fast_rk<float>(a, ws, st);
    if (rc != -3) return rc;
    if (kernel == 2) return -2;
  }
  int S = splits > 0 ? splits : decode_max_splits(a.U, a.N, a.M);
  if (S > ws.max_splits) S = ws.max_splits;
  DecodeParams p{a.U, a.G, a.d, a.r, a.N, a.M, a.q, a.Kc, a.V, a.R, a.dmu, a.Kt, a.Vt,
                 a.scale * kLog2e, a.out, ws.counters, ws.partials, nullptr, 0, a.pout,
                 a.nR > 0 ? a.nR : a.U, nullptr, nullptr, 0, a.Ms, a.nvu, a.ntu};
  size_t sm = ((size_t)a.G * a.d + (size_t)a.G * a.r + a.G + 2 * kGenWarps * a.G +
               (size_t)kGenWarps * a.G * a.d) * sizeof(float);
  dim3 grid(S, a.U);
  if (a.bf16) {
    cudaFuncSetAttribute(decode_generic_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    decode_generic_kernel<__nv_bfloat16><<<grid, kGenWarps * 32, sm, st>>>(p, S);
  } else {
    cudaFuncSetAttribute(decode_generic_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    decode_generic_kernel<float><<<grid, kGenWarps * 32, sm, st>>>(p, S);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// =====================================================================================
// merge of token-shard partial states (token-sharded decode for U < P):
//   out[u][g] = sum_p 2^(m_p - M) acc_p / sum_p 2^(m_p - M) l_p,   M = max_p m_p
// parts [P][U][G][d+2] (acc[d] | m | l, m in base-2 logit units), shards merged in order.
// =====================================================================================
__global__ void __launch_bounds__(128) merge_parts_kernel(int P, int UG, int d, const float* __restrict__ parts,
                                                          float* __restrict__ out) {
  const int ug = blockIdx.x;
  const size_t rec = (size_t)(d + 2), stride = (size_t)UG * rec;
  const float* base = parts + (size_t)ug * rec;
  float M = -CUDART_INF_F;
  for (int s = 0; s < P; ++s) M = fmaxf(M, base[s * stride + d]);
  float L = 0.f;
  for (int s = 0; s < P; ++s) {
    const float ms = base[s * stride + d];
    L = fmaf(base[s * stride + d + 1], ms == -CUDART_INF_F ? 0.f : fast_exp2(ms - M), L);
  }
  const float inv = 1.f / L;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float A = 0.f;
    for (int s = 0; s < P; ++s) {
      const float ms = base[s * stride + d];
      A = fmaf(base[s * stride + c], ms == -CUDART_INF_F ? 0.f : fast_exp2(ms - M), A);
    }
    out[(size_t)ug * d + c] = A * inv;
  }
}

int launch_merge_parts(int U, int G, int d, int P, const float* parts, float* out, cudaStream_t st) {
  merge_parts_kernel<<<U * G, 128, 0, st>>>(P, U * G, d, parts, out);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

void set_decode_trace(void* buf) { g_trace = static_cast<unsigned long long*>(buf); }
unsigned long long* decode_trace_buffer() { return g_trace; }
int decode_num_sms() { return num_sms(); }

}  // namespace rk
