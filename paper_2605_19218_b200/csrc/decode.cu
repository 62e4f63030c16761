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
//    byte of the compacted cache is read exactly once with no CTA-level barriers.  At
//    every unit boundary the warp flushes an online-softmax partial (m, l, acc[G][d]);
//    the last warp to finish a unit (atomic ticket) merges that unit's partials in slot
//    order (deterministic) and writes out, then re-arms the ticket (graph-replay safe).
//  * decode_generic_kernel (any d <= 256, any r, any G): one CTA per (unit, split),
//    plain loads, per-token online softmax.  Used for the toy shapes and fallbacks.
#include <cstdio>

#include "common.cuh"
#include "internal.h"

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
};

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
  const float* Ru = p.R + (size_t)u * d * r;
  for (int e = tid; e < G * r; e += blockDim.x) {
    const int g = e / r, k = e % r;
    float s = 0.f;
    for (int i = 0; i < d; ++i) s = fmaf(qs[g * d + i], Ru[(size_t)i * r + k], s);
    qt[e] = s * p.sl;
  }
  for (int g = w; g < G; g += kGenWarps) {
    float s = 0.f;
    if (p.dmu)
      for (int i = lane; i < d; i += 32) s = fmaf(qs[g * d + i], p.dmu[(size_t)u * d + i], s);
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
  for (int idx = w; idx < total; idx += kGenWarps) {
    const bool vis = idx < n1 - n0;
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
      krow = static_cast<const T*>(p.Kt) + ((size_t)u * p.M + t) * d;
      vrow = static_cast<const T*>(p.Vt) + ((size_t)u * p.M + t) * d;
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
      p.out[((size_t)u * G + g) * d + c] = A / L;
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
    p.out[((size_t)u * G + g) * d + c] = A / L;
  }
  if (tid == 0) p.counters[u] = 0u;
}

// =====================================================================================
// fast kernel: d = 128, warp-streaming with per-warp TMA bulk rings
// =====================================================================================
constexpr int kD = 128;

template <typename T, int RK, int G, int WARPS, int STAGES>
struct FastCfg {
  static constexpr int S = sizeof(T);
  static constexpr int CHB = 32;                       // bytes of a key row per lane
  static constexpr int CHN = CHB / S;                  // channels per lane chunk
  static constexpr int LPT_V = RK * S / CHB;           // lanes per visual token
  static constexpr int LPT_X = kD * S / CHB;           // lanes per text token
  static constexpr int TPS_V = 32 / LPT_V;             // visual tokens per step
  static constexpr int TPS_X = 32 / LPT_X;
  static constexpr int TT_V = (S == 2) ? 32 : 16;      // visual tile tokens
  static constexpr int STAGE = TT_V * (RK + kD) * S;   // bytes per stage
  static constexpr int TT_X = ((STAGE / (2 * kD * S)) / TPS_X) * TPS_X;
  static constexpr int NS_V = TT_V / TPS_V;
  static constexpr int NS_X = TT_X / TPS_X;
  static constexpr int VPL = kD / 32;                  // V dims per lane (4)
  // per-warp shared memory
  static constexpr int OFF_Q = STAGES * STAGE;                    // float [G][kD]
  static constexpr int OFF_QT = OFF_Q + G * kD * 4;              // float [G][RK]
  static constexpr int OFF_B = OFF_QT + G * RK * 4;              // float [G] (pad 4)
  static constexpr int OFF_BAR = (OFF_B + ((G + 3) / 4) * 16 + 7) / 8 * 8;
  static constexpr int WARP_SMEM = ((OFF_BAR + STAGES * 8) + 127) / 128 * 128;
  static constexpr int SMEM = WARPS * WARP_SMEM;
  static_assert(LPT_V >= 1 && LPT_V <= 32 && (32 % LPT_V) == 0, "bad RK");
  static_assert(TT_X >= TPS_X, "text tile too small");
  static_assert(TT_V % TPS_V == 0, "tile");
};

__device__ __forceinline__ long long range_start(long long T, int gw, int NW) {
  return T * gw / NW;
}
// warp whose range contains global token x
__device__ __forceinline__ int warp_of(long long x, long long T, int NW) {
  int g = (int)(x * NW / T);
  while (g + 1 < NW && range_start(T, g + 1, NW) <= x) ++g;
  while (g > 0 && range_start(T, g, NW) > x) --g;
  return g;
}

struct Tile {
  int u;      // unit
  int vis;    // 1 visual, 0 text
  int t;      // first token within the segment
  int tn;     // tokens in this tile
};

template <int TT_V, int TT_X>
__device__ __forceinline__ Tile tile_at(long long x, long long b, int N, int M) {
  const long long L = (long long)N + M;
  Tile tl;
  tl.u = (int)(x / L);
  const int off = (int)(x - (long long)tl.u * L);
  long long seg_end;
  if (off < N) {
    tl.vis = 1; tl.t = off;
    seg_end = (long long)tl.u * L + N;
    long long e = x + TT_V;
    if (e > seg_end) e = seg_end;
    if (e > b) e = b;
    tl.tn = (int)(e - x);
  } else {
    tl.vis = 0; tl.t = off - N;
    seg_end = (long long)(tl.u + 1) * L;
    long long e = x + TT_X;
    if (e > seg_end) e = seg_end;
    if (e > b) e = b;
    tl.tn = (int)(e - x);
  }
  return tl;
}

template <typename T>
__device__ __forceinline__ void unpack_chunk(const unsigned char* p, float* f);  // 32 bytes
template <>
__device__ __forceinline__ void unpack_chunk<__nv_bfloat16>(const unsigned char* p, float* f) {
  const uint4 a = *reinterpret_cast<const uint4*>(p);
  const uint4 b = *reinterpret_cast<const uint4*>(p + 16);
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) { f[2 * i] = bf16lo(w[i]); f[2 * i + 1] = bf16hi(w[i]); }
}
template <>
__device__ __forceinline__ void unpack_chunk<float>(const unsigned char* p, float* f) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 16);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

template <typename T>
__device__ __forceinline__ void load_v4(const unsigned char* p, float* f);
template <>
__device__ __forceinline__ void load_v4<__nv_bfloat16>(const unsigned char* p, float* f) {
  const uint2 a = *reinterpret_cast<const uint2*>(p);
  f[0] = bf16lo(a.x); f[1] = bf16hi(a.x); f[2] = bf16lo(a.y); f[3] = bf16hi(a.y);
}
template <>
__device__ __forceinline__ void load_v4<float>(const unsigned char* p, float* f) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
}

template <typename T, int RK, int G, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32, 1) decode_fast_kernel(DecodeParams p, int NW, int cmax) {
  using C = FastCfg<T, RK, G, WARPS, STAGES>;
  extern __shared__ __align__(128) unsigned char fsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * WARPS + w;
  if (gw >= NW) return;
  unsigned char* base = fsm + w * C::WARP_SMEM;
  float* qs = reinterpret_cast<float*>(base + C::OFF_Q);
  float* qts = reinterpret_cast<float*>(base + C::OFF_QT);
  float* bs = reinterpret_cast<float*>(base + C::OFF_B);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::OFF_BAR);

  const int N = p.N, M = p.M;
  const long long L = (long long)N + M;
  const long long Ttot = L * p.U;
  const long long a = range_start(Ttot, gw, NW), b = range_start(Ttot, gw + 1, NW);
  if (a >= b) return;

  const T* Kc = static_cast<const T*>(p.Kc);
  const T* V = static_cast<const T*>(p.V);
  const T* Kt = static_cast<const T*>(p.Kt);
  const T* Vt = static_cast<const T*>(p.Vt);
  const uint64_t pol = policy_evict_first();

  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  // ---------------- producer (lane 0): issue tile at cursor px into stage st
  long long px = a;
  auto issue = [&](int st) {
    const Tile tl = tile_at<C::TT_V, C::TT_X>(px, b, N, M);
    unsigned char* dst = base + st * C::STAGE;
    if (tl.vis) {
      const uint32_t kb = (uint32_t)tl.tn * RK * C::S, vb = (uint32_t)tl.tn * kD * C::S;
      mbar_arrive_expect_tx(&bar[st], kb + vb);
      bulk_g2s(dst, Kc + ((size_t)tl.u * N + tl.t) * RK, kb, &bar[st], pol);
      bulk_g2s(dst + C::TT_V * RK * C::S, V + ((size_t)tl.u * N + tl.t) * kD, vb, &bar[st], pol);
    } else {
      const uint32_t kb = (uint32_t)tl.tn * kD * C::S;
      mbar_arrive_expect_tx(&bar[st], 2 * kb);
      bulk_g2s(dst, Kt + ((size_t)tl.u * M + tl.t) * kD, kb, &bar[st], pol);
      bulk_g2s(dst + C::TT_X * kD * C::S, Vt + ((size_t)tl.u * M + tl.t) * kD, kb, &bar[st], pol);
    }
    px += tl.tn;
  };
  if (lane == 0)
    for (int s = 0; s < STAGES && px < b; ++s) issue(s);

  // ---------------- consumer state
  float m[G], l[G], acc[G][C::VPL];
  float qreg[C::CHN], xreg[C::CHN];  // used when G == 1
  int cur_u = -1;

  auto setup = [&](int u) {
    // q (fp32) -> smem; q~ = q R_r and b = q . dmu; then scale everything by sl
    const T* qg = static_cast<const T*>(p.q) + (size_t)u * G * kD;
    for (int e = lane; e < G * kD; e += 32) qs[e] = Elem<T>::to_f(qg[e]);
    __syncwarp();
    const float* Ru = p.R + (size_t)u * kD * RK;
    constexpr int KPL = (RK + 31) / 32;
    float qa[G][KPL];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int j = 0; j < KPL; ++j) qa[g][j] = 0.f;
#pragma unroll 4
    for (int i = 0; i < kD; ++i) {
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = lane + 32 * j;
        const float rv = (k < RK) ? __ldg(Ru + (size_t)i * RK + k) : 0.f;
#pragma unroll
        for (int g = 0; g < G; ++g) qa[g][j] = fmaf(qs[g * kD + i], rv, qa[g][j]);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = lane + 32 * j;
        if (k < RK) qts[g * RK + k] = qa[g][j] * p.sl;
      }
      float bb = 0.f;
      if (p.dmu) {
#pragma unroll
        for (int j = 0; j < kD / 32; ++j)
          bb = fmaf(qs[g * kD + lane + 32 * j], __ldg(p.dmu + (size_t)u * kD + lane + 32 * j), bb);
      }
      bb = warp_sum(bb);
      if (lane == 0) bs[g] = bb * p.sl;
    }
    __syncwarp();
    for (int e = lane; e < G * kD; e += 32) qs[e] *= p.sl;
    __syncwarp();
    if constexpr (G == 1) {
      const int cv = lane % C::LPT_V, cx = lane % C::LPT_X;
#pragma unroll
      for (int i = 0; i < C::CHN; ++i) {
        qreg[i] = qts[cv * C::CHN + i];
        xreg[i] = qs[cx * C::CHN + i];
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m[g] = -CUDART_INF_F;
      l[g] = 0.f;
#pragma unroll
      for (int k = 0; k < C::VPL; ++k) acc[g][k] = 0.f;
    }
  };

  auto flush = [&](int u) {
    const long long x0 = (long long)u * L, x1 = x0 + L - 1;
    const int first = warp_of(x0, Ttot, NW), last = warp_of(x1, Ttot, NW);
    const int count = last - first + 1;
    float lt[G];
#pragma unroll
    for (int g = 0; g < G; ++g) lt[g] = warp_sum(l[g]);
    if (count == 1) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float inv = 1.f / lt[g];
        float4 o = make_float4(acc[g][0] * inv, acc[g][1] * inv, acc[g][2] * inv, acc[g][3] * inv);
        *reinterpret_cast<float4*>(p.out + ((size_t)u * G + g) * kD + lane * 4) = o;
      }
      return;
    }
    // partial record: acc[kD] | m | l | pad[2]  (stride kRec floats, 16-byte aligned)
    constexpr int kRec = kD + 4;
    const int slot = gw - first;
    float* part = p.partials + ((size_t)u * cmax) * G * kRec;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float* dst = part + ((size_t)slot * G + g) * kRec;
      if (lane == 0) { dst[kD] = m[g]; dst[kD + 1] = lt[g]; }
      *reinterpret_cast<float4*>(dst + lane * 4) =
          make_float4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
    }
    __threadfence();
    __syncwarp();
    unsigned prev = 0;
    if (lane == 0) prev = atomicAdd(&p.counters[u], 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != (unsigned)(count - 1)) return;
    __threadfence();
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
      float Mx = -CUDART_INF_F;
      for (int s = 0; s < count; ++s) Mx = fmaxf(Mx, __ldcg(part + ((size_t)s * G + g) * kRec + kD));
      float Ls = 0.f, A[C::VPL] = {0.f, 0.f, 0.f, 0.f};
      for (int s = 0; s < count; ++s) {
        const float* src = part + ((size_t)s * G + g) * kRec;
        const float ms = __ldcg(src + kD);
        const float f = (ms == -CUDART_INF_F) ? 0.f : fast_exp2(ms - Mx);
        Ls = fmaf(__ldcg(src + kD + 1), f, Ls);
        const float4 v = __ldcg(reinterpret_cast<const float4*>(src + lane * 4));
        A[0] = fmaf(v.x, f, A[0]); A[1] = fmaf(v.y, f, A[1]);
        A[2] = fmaf(v.z, f, A[2]); A[3] = fmaf(v.w, f, A[3]);
      }
      const float inv = 1.f / Ls;
      *reinterpret_cast<float4*>(p.out + ((size_t)u * G + g) * kD + lane * 4) =
          make_float4(A[0] * inv, A[1] * inv, A[2] * inv, A[3] * inv);
    }
    if (lane == 0) p.counters[u] = 0u;
  };

  // ---------------- main loop over this warp's tiles
  long long cx = a;
  int j = 0;
  while (cx < b) {
    const Tile tl = tile_at<C::TT_V, C::TT_X>(cx, b, N, M);
    const int st = j % STAGES;
    const uint32_t ph = (uint32_t)((j / STAGES) & 1);
    if (tl.u != cur_u) {
      if (cur_u >= 0) flush(cur_u);
      setup(tl.u);
      cur_u = tl.u;
    }
    mbar_wait(&bar[st], ph);
    const unsigned char* kbuf = base + st * C::STAGE;
    if (tl.vis) {
      const unsigned char* vbuf = kbuf + C::TT_V * RK * C::S;
      float sc[G][C::NS_V];
      const int cv = lane % C::LPT_V, tv = lane / C::LPT_V;
#pragma unroll
      for (int s = 0; s < C::NS_V; ++s) {
        const int tok = s * C::TPS_V + tv;
        float kf[C::CHN];
        unpack_chunk<T>(kbuf + (size_t)tok * RK * C::S + cv * C::CHB, kf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float dsum = 0.f;
          if constexpr (G == 1) {
#pragma unroll
            for (int i = 0; i < C::CHN; ++i) dsum = fmaf(qreg[i], kf[i], dsum);
          } else {
            const float* qq = qts + g * RK + cv * C::CHN;
#pragma unroll
            for (int i = 0; i < C::CHN; i += 4) {
              const float4 q4 = *reinterpret_cast<const float4*>(qq + i);
              dsum = fmaf(q4.x, kf[i], dsum); dsum = fmaf(q4.y, kf[i + 1], dsum);
              dsum = fmaf(q4.z, kf[i + 2], dsum); dsum = fmaf(q4.w, kf[i + 3], dsum);
            }
          }
#pragma unroll
          for (int o = 1; o < C::LPT_V; o <<= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
          sc[g][s] = (tok < tl.tn) ? dsum + bs[g] : -CUDART_INF_F;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float tmax = sc[g][0];
#pragma unroll
        for (int s = 1; s < C::NS_V; ++s) tmax = fmaxf(tmax, sc[g][s]);
#pragma unroll
        for (int o = 16; o >= C::LPT_V; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        const float mn = fmaxf(m[g], tmax);
        const float alpha = fast_exp2(m[g] - mn);
        m[g] = mn;
        l[g] *= alpha;
#pragma unroll
        for (int k = 0; k < C::VPL; ++k) acc[g][k] *= alpha;
#pragma unroll
        for (int s = 0; s < C::NS_V; ++s) {
          const float pr = fast_exp2(sc[g][s] - mn);
          sc[g][s] = pr;
          if (cv == 0) l[g] += pr;
        }
      }
#pragma unroll
      for (int s = 0; s < C::NS_V; ++s) {
#pragma unroll 8
        for (int ii = 0; ii < C::TPS_V; ++ii) {
          const int tok = s * C::TPS_V + ii;
          if (tok >= tl.tn) break;
          float vf[C::VPL];
          load_v4<T>(vbuf + (size_t)tok * kD * C::S + lane * C::VPL * C::S, vf);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float pr = __shfl_sync(0xffffffffu, sc[g][s], ii * C::LPT_V);
#pragma unroll
            for (int k = 0; k < C::VPL; ++k) acc[g][k] = fmaf(pr, vf[k], acc[g][k]);
          }
        }
      }
    } else {
      const unsigned char* vbuf = kbuf + C::TT_X * kD * C::S;
      float sc[G][C::NS_X];
      const int cv = lane % C::LPT_X, tv = lane / C::LPT_X;
#pragma unroll
      for (int s = 0; s < C::NS_X; ++s) {
        const int tok = s * C::TPS_X + tv;
        float kf[C::CHN];
        unpack_chunk<T>(kbuf + (size_t)tok * kD * C::S + cv * C::CHB, kf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float dsum = 0.f;
          if constexpr (G == 1) {
#pragma unroll
            for (int i = 0; i < C::CHN; ++i) dsum = fmaf(xreg[i], kf[i], dsum);
          } else {
            const float* qq = qs + g * kD + cv * C::CHN;
#pragma unroll
            for (int i = 0; i < C::CHN; i += 4) {
              const float4 q4 = *reinterpret_cast<const float4*>(qq + i);
              dsum = fmaf(q4.x, kf[i], dsum); dsum = fmaf(q4.y, kf[i + 1], dsum);
              dsum = fmaf(q4.z, kf[i + 2], dsum); dsum = fmaf(q4.w, kf[i + 3], dsum);
            }
          }
#pragma unroll
          for (int o = 1; o < C::LPT_X; o <<= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
          sc[g][s] = (tok < tl.tn) ? dsum : -CUDART_INF_F;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float tmax = sc[g][0];
#pragma unroll
        for (int s = 1; s < C::NS_X; ++s) tmax = fmaxf(tmax, sc[g][s]);
#pragma unroll
        for (int o = 16; o >= C::LPT_X; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        const float mn = fmaxf(m[g], tmax);
        const float alpha = fast_exp2(m[g] - mn);
        m[g] = mn;
        l[g] *= alpha;
#pragma unroll
        for (int k = 0; k < C::VPL; ++k) acc[g][k] *= alpha;
#pragma unroll
        for (int s = 0; s < C::NS_X; ++s) {
          const float pr = fast_exp2(sc[g][s] - mn);
          sc[g][s] = pr;
          if (cv == 0) l[g] += pr;
        }
      }
#pragma unroll
      for (int s = 0; s < C::NS_X; ++s) {
#pragma unroll
        for (int ii = 0; ii < C::TPS_X; ++ii) {
          const int tok = s * C::TPS_X + ii;
          if (tok >= tl.tn) break;
          float vf[C::VPL];
          load_v4<T>(vbuf + (size_t)tok * kD * C::S + lane * C::VPL * C::S, vf);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float pr = __shfl_sync(0xffffffffu, sc[g][s], ii * C::LPT_X);
#pragma unroll
            for (int k = 0; k < C::VPL; ++k) acc[g][k] = fmaf(pr, vf[k], acc[g][k]);
          }
        }
      }
    }
    __syncwarp();
    // refill this stage with the tile STAGES ahead (the whole warp has consumed it)
    if (lane == 0 && px < b) {
      fence_proxy_async();
      issue(st);
    }
    cx += tl.tn;
    ++j;
  }
  if (cur_u >= 0) flush(cur_u);
}

// =====================================================================================
// host side
// =====================================================================================
constexpr int kFastWarps = 8;
constexpr int kFastStages = 2;

struct FastPlan {
  int NW;     // active warps
  int ctas;
  int cmax;   // max contributing warps per unit
};

static FastPlan fast_plan(int U, int N, int M, int warps) {
  FastPlan pl;
  const long long T = (long long)U * (N + M);
  long long nw = (long long)kNumSMs * warps;
  const long long by_size = (T + 63) / 64;  // at least 64 tokens per warp
  if (by_size < nw) nw = by_size;
  if (nw < 1) nw = 1;
  pl.NW = (int)nw;
  pl.ctas = (pl.NW + warps - 1) / warps;
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

size_t decode_ws_layout(int U, int G, int d, int N, int M, void* base, DecodeWs* ws) {
  const FastPlan pl = fast_plan(U, N, M, kFastWarps);  // worst case: most warps per unit
  int smax = decode_max_splits(U, N, M);
  if (smax < 64) {
    // explicit splits (rotatek_decode_attn_ex) may ask for up to 64
    smax = 64;
  }
  size_t gen = (size_t)U * G * smax * (d + 2) * 4;
  size_t fast = (size_t)U * pl.cmax * G * (d + 4) * 4;
  size_t part = gen > fast ? gen : fast;
  char* b = static_cast<char*>(base);
  size_t off = 0;
  DecodeWs w;
  w.counters = (uint32_t*)(b ? b + off : nullptr);
  off += al256((size_t)U * 4);
  w.partials = (float*)(b ? b + off : nullptr);
  off += al256(part);
  w.max_splits = smax;
  if (ws) *ws = w;
  return off;
}

template <typename T, int RK, int G>
constexpr int fast_warps() {
  constexpr int per = FastCfg<T, RK, G, 1, kFastStages>::WARP_SMEM;
  constexpr int w = (227 * 1024) / per;
  return w > kFastWarps ? kFastWarps : w;
}

template <typename T, int RK, int G>
static int launch_fast_t(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  constexpr int WARPS = fast_warps<T, RK, G>();
  using C = FastCfg<T, RK, G, WARPS, kFastStages>;
  const FastPlan pl = fast_plan(a.U, a.N, a.M, WARPS);
  DecodeParams p{a.U, a.G, a.d, a.r, a.N, a.M, a.q, a.Kc, a.V, a.R, a.dmu, a.Kt, a.Vt,
                 a.scale * kLog2e, a.out, ws.counters, ws.partials};
  auto kern = decode_fast_kernel<T, RK, G, WARPS, kFastStages>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  kern<<<pl.ctas, WARPS * 32, C::SMEM, st>>>(p, pl.NW, pl.cmax);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T>
static int launch_fast_rk(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  if (a.G == 1) {
    switch (a.r) {
      case 16: return launch_fast_t<T, 16, 1>(a, ws, st);
      case 32: return launch_fast_t<T, 32, 1>(a, ws, st);
      case 64: return launch_fast_t<T, 64, 1>(a, ws, st);
      case 128: return launch_fast_t<T, 128, 1>(a, ws, st);
    }
  } else if (a.G == 7) {
    switch (a.r) {
      case 16: return launch_fast_t<T, 16, 7>(a, ws, st);
      case 32: return launch_fast_t<T, 32, 7>(a, ws, st);
      case 64: return launch_fast_t<T, 64, 7>(a, ws, st);
      case 128: return launch_fast_t<T, 128, 7>(a, ws, st);
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

int launch_decode(const DecodeArgs& a, const DecodeWs& ws, int splits, int kernel, cudaStream_t st) {
  const bool fast_ok = fast_supported(a);
  if (kernel == 2 && !fast_ok) return -2;
  if ((kernel == 0 && fast_ok && splits <= 0) || kernel == 2) {
    return a.bf16 ? launch_fast_rk<__nv_bfloat16>(a, ws, st) : launch_fast_rk<float>(a, ws, st);
  }
  int S = splits > 0 ? splits : decode_max_splits(a.U, a.N, a.M);
  if (S > ws.max_splits) S = ws.max_splits;
  DecodeParams p{a.U, a.G, a.d, a.r, a.N, a.M, a.q, a.Kc, a.V, a.R, a.dmu, a.Kt, a.Vt,
                 a.scale * kLog2e, a.out, ws.counters, ws.partials};
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

}  // namespace rk
