// decode_steal.cuh -- the streaming decode with work stealing (included by decode.cu after
// decode_fast.cuh; same tiles, rotation table, tile_compute and merges).
//
// Why: with static equal token ranges the warps' finish times spread by 10-30 us (per-warp
// %globaltimer traces), and the spread follows the ADDRESS RANGE (finish times correlate
// 0.65-0.7 between launches, also with the CTA->SM mapping rotated), so no static split
// balances it.  Here every warp owns its equal range but CLAIMS it C tokens at a time from
// a global descriptor; a warp that runs dry steals the back half of the largest remaining
// range.  The tail then ends within about one claim of the mean finish time.
//
//   desc[w] (u64) = end << 32 | next : warp w's unclaimed tokens [next, end) (global token
//                   index x = u*(N+M) + t).  The owner claims with atomicAdd(desc, C) (one
//                   claim ahead, so its latency hides behind a tile); a thief CASes end down.
//   runs          : maximal contiguous token intervals one warp processes within one unit.
//                   A run covering a whole unit writes out directly; otherwise it takes a
//                   partial slot (atomicAdd nslot[u]) and adds its token count to ntok[u]
//                   (acq_rel); the run that completes the unit's N+M tokens merges the slots
//                   and re-arms both counters.  Merge order = slot order (timing dependent:
//                   results are reproducible to fp32 re-association, not bit for bit).
//   stolen units  : a unit outside the CTA's query table is rotated by the thief itself
//                   (rotate_cols, one round trip) into the warp's private entry.

template <typename T, int RK, int G, int WARPS, int STAGES, int TTV>
struct StealCfg : FastCfg<T, RK, G, WARPS, STAGES, TTV> {
  using B = FastCfg<T, RK, G, WARPS, STAGES, TTV>;
  static constexpr int OFF_PRIV = B::SMEM;                     // per-warp private QEnt (thieves)
  static constexpr int SMEM = OFF_PRIV + WARPS * B::ENT;
};

template <typename T, int RK, int G, int WARPS, int STAGES, int TTV, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) decode_steal_kernel(DecodeParams p, int NW, int cmax,
                                                                        int claim, int smin) {
  using C = StealCfg<T, RK, G, WARPS, STAGES, TTV>;
  constexpr int NACC = C::NACC;
  extern __shared__ __align__(128) unsigned char fsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * p.aw + w;
  unsigned char* base = fsm + w * C::WARP_SMEM;
  float* qs = reinterpret_cast<float*>(base + C::OFF_Q);
  float* pbuf = reinterpret_cast<float*>(base + C::OFF_P);
  unsigned char* tab = fsm + C::OFF_TAB;
  unsigned char* priv = fsm + C::OFF_PRIV + w * C::ENT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::OFF_BAR);

  const int N = p.N, M = p.M;
  const long long L = (long long)N + M;
  const long long Ttot = L * p.U;
  RK_TRACE(0, gtime());
  int uA, nu;
  const Split sp{Ttot, L, NW, N};
  cta_units(sp, p.aw, blockIdx.x, uA, nu);
  const long long a0 = sp.start(gw), b0 = sp.start(gw + 1);
  const bool active = w < p.aw && gw < NW && a0 < b0;

  const T* Kc = static_cast<const T*>(p.Kc);
  const T* V = static_cast<const T*>(p.V);
  const T* Kt = static_cast<const T*>(p.Kt);
  const T* Vt = static_cast<const T*>(p.Vt);
  const uint64_t pol = policy_evict_first();

  if (active && lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  StealSched sched{p.desc, gw, NW, claim, smin, lane};
  sched.init(active, a0, b0);
  __syncwarp();
  auto next_tile = [&](Tile& tl, uint32_t& x) { return sched.template next<C::TT_V, C::TT_X>(tl, x, N, M); };
  auto issue = [&](int st, const Tile& tl) {
    if (lane != 0) return;
    unsigned char* dst = base + st * C::STAGE;
    if (tl.vis) {
      const uint32_t kb = (uint32_t)tl.tn * RK * C::S, vb = (uint32_t)tl.tn * kD * C::S;
      mbar_arrive_expect_tx(&bar[st], kb + vb);
      bulk_g2s(dst, Kc + ((size_t)tl.u * N + tl.t) * RK, kb, &bar[st], pol);
      bulk_g2s(dst + C::TT_V * RK * C::S, V + ((size_t)tl.u * N + tl.t) * kD, vb, &bar[st], pol);
    } else {
      const uint32_t kb = (uint32_t)tl.tn * kD * C::S;
      mbar_arrive_expect_tx(&bar[st], 2 * kb);
      bulk_g2s(dst, Kt + ((size_t)tl.u * p.Ms + tl.t) * kD, kb, &bar[st], pol);
      bulk_g2s(dst + C::TT_X * kD * C::S, Vt + ((size_t)tl.u * p.Ms + tl.t) * kD, kb, &bar[st], pol);
    }
  };

  pdl_launch_dependents();
  rotate_cta<T, RK, G, WARPS, C::ENT>(p, uA, nu, w, lane, tab);  // query table, then tiles
  RK_TRACE(1, gtime());
  if (!active) return;

  Tile md[STAGES];
  uint32_t mx[STAGES];
  bool live[STAGES];
#pragma unroll
  for (int s = 0; s < STAGES; ++s) {
    live[s] = next_tile(md[s], mx[s]);
    if (live[s]) issue(s, md[s]);
  }

  // ---------------- consumer state (one run at a time)
  float m[G], l[G], acc[NACC][G][4];
  float qreg[C::CHN], xreg[C::CHN];
  int run_u = -1;
  uint32_t run_s = 0, run_e = 0;
  const float* qts = nullptr;
  const float* bs = nullptr;

  auto setup = [&](int u) {
    unsigned char* ent;
    if (u >= uA && u < uA + nu) {
      ent = tab + (u - uA) * C::ENT;
    } else {  // stolen work outside the CTA's table: rotate it here
      __syncwarp();
      rotate_cols<T, RK, RK, G>(p, u, 0, lane, priv);
      __syncwarp();
      ent = priv;
    }
    using E = QEnt<T, RK, G>;
    qts = reinterpret_cast<const float*>(ent);
    bs = reinterpret_cast<const float*>(ent + E::OFF_B);
    const T* qe = reinterpret_cast<const T*>(ent + E::OFF_Q);
    if constexpr (G == 1) {
      const int cv = lane % C::LPT_V, cx = lane % C::LPT_X;
#pragma unroll
      for (int i = 0; i < C::CHN; ++i) {
        qreg[i] = qts[cv * C::CHN + i];
        xreg[i] = Elem<T>::to_f(qe[cx * C::CHN + i]) * p.sl;
      }
    } else {
      for (int e = lane; e < G * kD; e += 32) qs[e] = Elem<T>::to_f(qe[e]) * p.sl;
      __syncwarp();
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m[g] = -CUDART_INF_F;
      l[g] = 0.f;
#pragma unroll
      for (int aa = 0; aa < NACC; ++aa)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[aa][g][k] = 0.f;
    }
  };

  auto flush = [&]() {
    const int u = run_u;
    float lt[G], A[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      lt[g] = warp_sum(l[g]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        A[g][k] = acc[0][g][k];
#pragma unroll
        for (int aa = 1; aa < NACC; ++aa) A[g][k] += acc[aa][g][k];
      }
    }
    const uint32_t len = run_e - run_s;
    if ((long long)len == L) {  // this run is the whole unit
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (p.pout) {
          float* po = p.pout + ((size_t)u * G + g) * (kD + 2);
#pragma unroll
          for (int k = 0; k < 4; ++k) po[lane * 4 + k] = A[g][k];
          if (lane == 0) { po[kD] = m[g]; po[kD + 1] = lt[g]; }
        } else {
          const float inv = 1.f / lt[g];
          *reinterpret_cast<float4*>(p.out + ((size_t)u * G + g) * kD + lane * 4) =
              make_float4(A[g][0] * inv, A[g][1] * inv, A[g][2] * inv, A[g][3] * inv);
        }
      }
      return;
    }
    constexpr int kRec = kD + 4;
    unsigned slot = 0;
    if (lane == 0) slot = atomicAdd(&p.nslot[u], 1u);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (slot >= (unsigned)cmax) __trap();  // host bound on runs per unit violated
    float* part = p.partials + ((size_t)u * cmax) * G * kRec;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float* dst = part + ((size_t)slot * G + g) * kRec;
      if (lane == 0) { dst[kD] = m[g]; dst[kD + 1] = lt[g]; }
      *reinterpret_cast<float4*>(dst + lane * 4) = make_float4(A[g][0], A[g][1], A[g][2], A[g][3]);
    }
    __syncwarp();
    unsigned prev = 0;
    if (lane == 0) prev = atom_add_acq_rel_gpu(&p.counters[u], len);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if ((long long)prev + len != L) return;
    unsigned count = 0;
    if (lane == 0) count = *reinterpret_cast<volatile unsigned*>(&p.nslot[u]);
    count = __shfl_sync(0xffffffffu, count, 0);
    merge_unit<G>(part, (int)count, p.out + (size_t)u * G * kD, lane,
                  p.pout ? p.pout + (size_t)u * G * (kD + 2) : nullptr);
    if (lane == 0) { p.counters[u] = 0u; p.nslot[u] = 0u; }
  };

  // ---------------- main loop: tiles in issue order, one ring slot at a time
  int j = 0;
  while (true) {
    const int st = j % STAGES;
    if (!live[st]) break;
    const Tile tl = md[st];
    const uint32_t x = mx[st];
    if (tl.u != run_u || x != run_e) {  // new run: unit change or a jump (stolen work)
      if (run_u >= 0) flush();
      setup(tl.u);
      run_u = tl.u;
      run_s = x;
    }
    run_e = x + (uint32_t)tl.tn;
    mbar_wait(&bar[st], (uint32_t)((j / STAGES) & 1));
    if (j == 0) RK_TRACE(2, gtime());
    const unsigned char* kbuf = base + st * C::STAGE;
    const int tv = valid_tn(p, tl.u, tl.vis, tl.t, tl.tn);  // variable lengths: mask padding
    if (tv == 0) {
    } else if (tl.vis) {
      const unsigned char* vbuf = kbuf + C::TT_V * RK * C::S;
      if (tv == C::TT_V)
        tile_compute<T, RK, C::TT_V, G, NACC, true, true>(kbuf, vbuf, tv, qts, qreg, bs, pbuf,
                                                          m, l, acc, lane);
      else
        tile_compute<T, RK, C::TT_V, G, NACC, false, true>(kbuf, vbuf, tv, qts, qreg, bs, pbuf,
                                                           m, l, acc, lane);
    } else {
      const unsigned char* vbuf = kbuf + C::TT_X * kD * C::S;
      if (tv == C::TT_X)
        tile_compute<T, kD, C::TT_X, G, NACC, true, false>(kbuf, vbuf, tv, qs, xreg, bs, pbuf,
                                                           m, l, acc, lane);
      else
        tile_compute<T, kD, C::TT_X, G, NACC, false, false>(kbuf, vbuf, tv, qs, xreg, bs, pbuf,
                                                            m, l, acc, lane);
    }
    // refill this slot (the whole warp has consumed it)
    live[st] = next_tile(md[st], mx[st]);
    if (live[st]) {
      if (lane == 0) fence_proxy_async();
      issue(st, md[st]);
    }
    ++j;
  }
  RK_TRACE(3, gtime());
  if (run_u >= 0) flush();
  RK_TRACE(4, gtime());
  RK_TRACE(5, (unsigned long long)j);
  RK_TRACE(6, (unsigned long long)nu);
}
