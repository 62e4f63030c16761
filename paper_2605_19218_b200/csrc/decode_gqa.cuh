// decode_gqa.cuh -- tensor-core decode for grouped-query attention (G query heads per KV
// unit, 2 <= G <= 8; d = 128; r in {32, 64}; bf16 cache).  Included by decode.cu.
//
// Same warp-streaming decomposition as decode_fast_kernel (one contiguous token range per
// warp, per-warp TMA stage, unit-boundary partials merged by the last contributor), but
// the arithmetic runs on the tensor cores with mma.sync.m16n8k16 (bf16 in, fp32 accumulate):
//   scores  S[16 x 8] = A[16 x 16] . K~^T   A rows 0..G-1 = q~ rounded to bf16 (hi),
//                                           rows 8..8+G-1 = q~ - hi rounded (lo); the hi and
//                                           lo partial scores land in the same thread and are
//                                           summed, so q~ enters with ~16 significant bits;
//   P.V     O[16 x 8] = P[16 x 16] . V      P rows 0..7 = bf16(p), rows 8..15 = p - bf16(p);
// K~ and V tiles are brought by tensor-map TMA (cp.async.bulk.tensor, 64/128-byte swizzle)
// so that ldmatrix (and ldmatrix.trans for V) reads them without bank conflicts; tokens past
// the end of a unit are zero-filled by TMA, tokens past the end of the warp's range are masked.
// tcgen05 is not used here: with M = 2G <= 16 useful rows its 64/128-row tiles would waste
// 4-8x of the tensor pipe, while the kernel is HBM-bound (~7 flop/byte).


template <int RK, int G, int WARPS, int TTV = 64, int STAGES = 1, bool STEAL = false>
struct GqaCfg {
  static constexpr int TT = TTV;                    // visual tile tokens
  static constexpr int KB = TT * RK * 2;            // K~ box bytes
  static constexpr int VH = TT * 128;               // one 64-channel V half
  static constexpr int STAGE = (KB + 2 * VH + 1023) / 1024 * 1024;
  static constexpr int TX = (STAGE / 512) / 16 * 16;  // text tile tokens (4 halves fit a stage)
  static constexpr int XH = TX * 128;               // one 64-channel text half
  static constexpr int NSTG = STAGES;
  static constexpr int OFF_BAR = NSTG * STAGE;
  static constexpr int WARP_SMEM = (OFF_BAR + 8 * NSTG + 1023) / 1024 * 1024;
  static constexpr int CAP = 8;                                // CTA query table (units)
  static constexpr int ENT = QEnt<__nv_bfloat16, RK, G>::BYTES;
  static constexpr int OFF_TAB = WARPS * WARP_SMEM;
  static constexpr int OFF_PRIV = OFF_TAB + CAP * ENT;         // per-warp QEnt for stolen units
  static constexpr int SMEM = OFF_PRIV + (STEAL ? WARPS * ENT : 0) + 1024;  // + alignment slack
  static_assert(STAGE >= 4 * XH && TX >= 16, "text tile must fit the stage");
  static_assert(TT % 16 == 0 && KB % 1024 == 0, "tile");
  static_assert(RK == 32 || RK == 64, "rank");
  static_assert(G >= 1 && G <= 8, "group");
};

struct GqaMaps {
  CUtensorMap kc, v, kt, vt;
};

// static ranges: the warp's equal share [a, b), tile by tile
struct StaticSched {
  long long px, b;
  template <int TTV, int TTX>
  __device__ __forceinline__ bool next(Tile& tl, uint32_t& x, int N, int M) {
    if (px >= b) return false;
    tl = tile_at<TTV, TTX>(px, b, N, M);
    x = (uint32_t)px;
    px += tl.tn;
    return true;
  }
};

// STEAL: the tile source is StealSched (decode_steal.cuh describes the protocol)
template <int RK, int G, int WARPS, int TTV, int STAGES, bool STEAL>
__global__ void __launch_bounds__(WARPS * 32, 1) decode_gqa_kernel(const __grid_constant__ GqaMaps maps,
                                                                   DecodeParams p, int NW, int cmax,
                                                                   int claim) {
  using C = GqaCfg<RK, G, WARPS, TTV, STAGES, STEAL>;
  constexpr int NKS = RK / 16;  // score k-steps
  extern __shared__ unsigned char gsm_raw[];
  unsigned char* gsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * p.aw + w;
  unsigned char* base = gsm + w * C::WARP_SMEM;
  unsigned char* tab = gsm + C::OFF_TAB;
  unsigned char* priv = gsm + C::OFF_PRIV + w * C::ENT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::OFF_BAR);
  const uint32_t sbase = smem_u32(base);

  const int N = p.N, M = p.M;
  const long long L = (long long)N + M;
  const long long Ttot = L * p.U;
  RK_TRACE(0, gtime());
  int uA, nu;
  const Split sp{Ttot, L, NW, N};
  cta_units(sp, p.aw, blockIdx.x, uA, nu);
  const long long a = sp.start(gw), b = sp.start(gw + 1);
  const bool active = w < p.aw && gw < NW && a < b;
  const uint64_t pol = policy_evict_first();
  if (active && lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    tc::prefetch_tmap(&maps.kc);
    tc::prefetch_tmap(&maps.v);
    if (M > 0) {
      tc::prefetch_tmap(&maps.kt);
      tc::prefetch_tmap(&maps.vt);
    }
  }
  __syncwarp();

  // tile source: static equal ranges, or work stealing
  using Sched = typename std::conditional<STEAL, StealSched, StaticSched>::type;
  Sched sched;
  if constexpr (STEAL) {
    sched = StealSched{p.desc, gw, NW, claim, claim, lane};
    sched.init(active, a, b);
  } else {
    sched = StaticSched{a, b};
  }
  auto next_tile = [&](Tile& tl, uint32_t& x) { return sched.template next<C::TT, C::TX>(tl, x, N, M); };
  auto issue = [&](int st, const Tile& tl) {
    if (lane != 0) return;
    unsigned char* dst = base + st * C::STAGE;
    uint64_t* bb = &bar[st];
    if (tl.vis) {
      mbar_arrive_expect_tx(bb, C::KB + 2 * C::VH);
      tc::tma_load_3d(dst, &maps.kc, 0, tl.t, tl.u, bb, pol);
      tc::tma_load_3d(dst + C::KB, &maps.v, 0, tl.t, tl.u, bb, pol);
      tc::tma_load_3d(dst + C::KB + C::VH, &maps.v, 64, tl.t, tl.u, bb, pol);
    } else {
      mbar_arrive_expect_tx(bb, 4 * C::XH);
      tc::tma_load_3d(dst, &maps.kt, 0, tl.t, tl.u, bb, pol);
      tc::tma_load_3d(dst + C::XH, &maps.kt, 64, tl.t, tl.u, bb, pol);
      tc::tma_load_3d(dst + 2 * C::XH, &maps.vt, 0, tl.t, tl.u, bb, pol);
      tc::tma_load_3d(dst + 3 * C::XH, &maps.vt, 64, tl.t, tl.u, bb, pol);
    }
  };
  pdl_launch_dependents();
  Tile md[STAGES];
  uint32_t mx[STAGES];
  bool livest[STAGES];
  auto first_tiles = [&] {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      livest[s] = next_tile(md[s], mx[s]);
      if (livest[s]) issue(s, md[s]);
    }
  };
  // query table, then tiles -- or, when launched overlapped with the preceding kernel, the
  // first tiles (cache bytes are complete by contract) while it finishes, then the table
  if (p.overlap && active) first_tiles();
  rotate_cta<__nv_bfloat16, RK, G, WARPS, C::ENT>(p, uA, nu, w, lane, tab);
  RK_TRACE(1, gtime());
  if (!active) return;
  if (!p.overlap) first_tiles();

  const int g = lane >> 2, c = lane & 3;
  const bool live = g < G;
  uint32_t aq[NKS][4];   // q~ hi/lo A fragments
  uint32_t ax[8][4];     // q hi/lo A fragments (text)
  float bg = 0.f;
  float m = -CUDART_INF_F, l = 0.f;
  float acc[16][4];
  int cur_u = -1;
  uint32_t run_s = 0, run_e = 0;

  auto setup = [&](int u) {
    // q~ = q R_r, b = q . dmu and q of the unit's G heads from the CTA's rotation table (or,
    // for stolen work outside it, rotated here into the warp's private entry)
    using E = QEnt<__nv_bfloat16, RK, G>;
    const unsigned char* ent = tab + (u - uA) * C::ENT;
    if constexpr (STEAL) {
      if (u < uA || u >= uA + nu) {
        __syncwarp();
        rotate_cols<__nv_bfloat16, RK, RK, G>(p, u, 0, lane, priv);
        __syncwarp();
        ent = priv;
      }
    }
    const float* qts = reinterpret_cast<const float*>(ent);
    const float* bs = reinterpret_cast<const float*>(ent + E::OFF_B);
    // A fragments straight from global memory (all loads independent): row g holds the
    // bf16 "hi" part, row g + 8 the "lo" remainder; k columns 2c, 2c+1 and 8+2c, 9+2c.
    const int gl = live ? g : 0;
    const float2* t2 = reinterpret_cast<const float2*>(qts + gl * RK);
    const __nv_bfloat162* q2 =
        reinterpret_cast<const __nv_bfloat162*>(ent + E::OFF_Q) + gl * (kD / 2);
    float2 tq[NKS][2];
    __nv_bfloat162 xq[8][2];
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk) {
      tq[kk][0] = t2[8 * kk + c];
      tq[kk][1] = t2[8 * kk + 4 + c];
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      xq[kk][0] = q2[8 * kk + c];
      xq[kk][1] = q2[8 * kk + 4 + c];
    }
    const float bq = bs[gl];
    const float z = live ? 1.f : 0.f;
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk) {
      gqa::split2(z * tq[kk][0].x, z * tq[kk][0].y, aq[kk][0], aq[kk][1]);
      gqa::split2(z * tq[kk][1].x, z * tq[kk][1].y, aq[kk][2], aq[kk][3]);
    }
    const float zs = z * p.sl;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const float2 lo = __bfloat1622float2(xq[kk][0]), hi = __bfloat1622float2(xq[kk][1]);
      gqa::split2(zs * lo.x, zs * lo.y, ax[kk][0], ax[kk][1]);
      gqa::split2(zs * hi.x, zs * hi.y, ax[kk][2], ax[kk][3]);
    }
    bg = z * bq;
    m = -CUDART_INF_F;
    l = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][e] = 0.f;
  };

  // online softmax over NB n-blocks of scores s[NB][2] (row g), then P.V from V halves
  auto softmax_pv = [&](auto nb_tag, float (&s)[decltype(nb_tag)::value][2], uint32_t v0, uint32_t vhalf) {
    constexpr int NB = decltype(nb_tag)::value;
    float tmax = -CUDART_INF_F;
#pragma unroll
    for (int j = 0; j < NB; ++j) tmax = fmaxf(tmax, fmaxf(s[j][0], s[j][1]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float mn = live ? fmaxf(m, tmax) : 0.f;
    const float alpha = live ? fast_exp2(m - mn) : 0.f;
    m = mn;
    l *= alpha;
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][e] *= alpha;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      s[j][0] = live ? fast_exp2(s[j][0] - mn) : 0.f;
      s[j][1] = live ? fast_exp2(s[j][1] - mn) : 0.f;
      l += s[j][0] + s[j][1];
    }
#pragma unroll
    for (int kt = 0; kt < NB / 2; ++kt) {
      uint32_t pa[4];
      gqa::split2(s[2 * kt][0], s[2 * kt][1], pa[0], pa[1]);
      gqa::split2(s[2 * kt + 1][0], s[2 * kt + 1][1], pa[2], pa[3]);
      const int mid = lane >> 3, r8 = lane & 7;
      const uint32_t tok = 16 * kt + r8 + 8 * (mid & 1);
#pragma unroll
      for (int cbp = 0; cbp < 8; ++cbp) {
        const uint32_t cb = 2 * cbp + (mid >> 1);
        const uint32_t addr = v0 + (cb >> 3) * vhalf + gqa::swz<128>(tok, cb & 7);
        uint32_t b0, b1, b2, b3;
        gqa::ldsm_x4_t(addr, b0, b1, b2, b3);
        gqa::mma16816(acc[2 * cbp], pa, b0, b1);
        gqa::mma16816(acc[2 * cbp + 1], pa, b2, b3);
      }
    }
  };

  // the last arrival at a unit's ticket merges its partials
  auto arrive = [&](int u, int count) {
    constexpr int kRec = kD + 4;
    __syncwarp();
    unsigned prev = 0;
    if (lane == 0) prev = atom_add_acq_rel_gpu(&p.counters[u], 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != (unsigned)(count - 1)) return;
    merge_unit<G>(p.partials + ((size_t)u * cmax) * G * kRec, count, p.out + (size_t)u * G * kD, lane,
                  p.pout ? p.pout + (size_t)u * G * (kD + 2) : nullptr);
    if (lane == 0) p.counters[u] = 0u;
  };
  auto flush = [&](int u) {
    int count, first = 0;
    if constexpr (STEAL) {
      count = (long long)(run_e - run_s) == L ? 1 : 0;  // 0: a partial run (dynamic slot)
    } else {
      const long long x0 = (long long)u * L, x1 = x0 + L - 1;
      first = sp.warp_of(x0);
      count = sp.warp_of(x1) - first + 1;
    }
    float lt = l + __shfl_xor_sync(0xffffffffu, l, 1);
    lt += __shfl_xor_sync(0xffffffffu, lt, 2);
    constexpr int kRec = kD + 4;
    if (count == 1 && p.pout) {
      if (live) {
        float* po = p.pout + ((size_t)u * G + g) * (kD + 2);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          po[8 * j + 2 * c] = acc[j][0] + acc[j][2];
          po[8 * j + 2 * c + 1] = acc[j][1] + acc[j][3];
        }
        if (c == 0) { po[kD] = m; po[kD + 1] = lt; }
      }
      return;
    }
    if (count == 1) {
      if (live) {
        const float inv = 1.f / lt;
        float* o = p.out + ((size_t)u * G + g) * kD + 2 * c;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          *reinterpret_cast<float2*>(o + 8 * j) =
              make_float2((acc[j][0] + acc[j][2]) * inv, (acc[j][1] + acc[j][3]) * inv);
      }
      return;
    }
    int slot = gw - first;
    if constexpr (STEAL) {
      unsigned sl = 0;
      if (lane == 0) sl = atomicAdd(&p.nslot[u], 1u);
      slot = (int)__shfl_sync(0xffffffffu, sl, 0);
      if (slot >= cmax) __trap();  // host bound on runs per unit violated
    }
    float* part = p.partials + ((size_t)u * cmax) * G * kRec;
    if (live) {
      float* dst = part + ((size_t)slot * G + g) * kRec;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        *reinterpret_cast<float2*>(dst + 8 * j + 2 * c) = make_float2(acc[j][0] + acc[j][2], acc[j][1] + acc[j][3]);
      if (c == 0) { dst[kD] = m; dst[kD + 1] = lt; }
    }
    if constexpr (STEAL) {
      // token ticket: the run that completes the unit's N+M tokens merges every slot
      __syncwarp();
      const unsigned len = run_e - run_s;
      unsigned prev = 0;
      if (lane == 0) prev = atom_add_acq_rel_gpu(&p.counters[u], len);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if ((long long)prev + len != L) return;
      unsigned cnt = 0;
      if (lane == 0) cnt = *reinterpret_cast<volatile unsigned*>(&p.nslot[u]);
      cnt = __shfl_sync(0xffffffffu, cnt, 0);
      merge_unit<G>(part, (int)cnt, p.out + (size_t)u * G * kD, lane,
                    p.pout ? p.pout + (size_t)u * G * (kD + 2) : nullptr);
      if (lane == 0) { p.counters[u] = 0u; p.nslot[u] = 0u; }
    } else {
      arrive(u, count);
    }
  };

  // rows [t0, t1) of both 64-channel V halves (128-byte rows; the swizzle permutes chunks
  // within a row only) set to zero: masked tokens get p = 0, and 0 * (padding NaN/Inf) would
  // still poison the tensor-core P.V.
  auto zero_rows = [&](unsigned char* v0, int half, int t0, int t1) {
    const int n = (t1 - t0) * 8;  // 16-byte chunks per half
    for (int i = lane; i < 2 * n; i += 32) {
      const int h = i >= n, k = i - h * n;
      reinterpret_cast<uint4*>(v0 + h * half + t0 * 128)[k] = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async();  // every writer: ordered before the stage's next TMA fill
    __syncwarp();
  };

  using NbV = std::integral_constant<int, C::TT / 8>;
  using NbX = std::integral_constant<int, C::TX / 8>;

  int j = 0;
  while (true) {
    const int st = j % STAGES;
    if (!livest[st]) break;
    const Tile tl = md[st];
    const uint32_t x = mx[st];
    if (tl.u != cur_u || x != run_e) {  // new run: unit change (or a jump to stolen work)
      if (cur_u >= 0) flush(cur_u);
      setup(tl.u);
      cur_u = tl.u;
      run_s = x;
    }
    run_e = x + (uint32_t)tl.tn;
    mbar_wait(&bar[st], (uint32_t)((j / STAGES) & 1));
    if (j == 0) RK_TRACE(2, gtime());
    const uint32_t sb = sbase + st * C::STAGE;
    const int mid = lane >> 3, r8 = lane & 7;
    const int tv = valid_tn(p, tl.u, tl.vis, tl.t, tl.tn);  // variable lengths: mask padding
    if (tv == 0) {
    } else if (tl.vis) {
      float s[NbV::value][2];
#pragma unroll
      for (int nb = 0; nb < NbV::value; ++nb) {
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t row = 8 * nb + r8;
#pragma unroll
        for (int kp = 0; kp < RK / 32; ++kp) {
          uint32_t b0, b1, b2, b3;
          gqa::ldsm_x4(sb + gqa::swz<RK * 2>(row, 4 * kp + mid), b0, b1, b2, b3);
          gqa::mma16816(d, aq[2 * kp], b0, b1);
          gqa::mma16816(d, aq[2 * kp + 1], b2, b3);
        }
        const int t0 = 8 * nb + 2 * c;
        s[nb][0] = (t0 < tv) ? d[0] + d[2] + bg : -CUDART_INF_F;
        s[nb][1] = (t0 + 1 < tv) ? d[1] + d[3] + bg : -CUDART_INF_F;
      }
      if (tv < C::TT) zero_rows(base + st * C::STAGE + C::KB, C::VH, tv, C::TT);
      softmax_pv(NbV{}, s, sb + C::KB, C::VH);
    } else {
      float s[NbX::value][2];
#pragma unroll
      for (int nb = 0; nb < NbX::value; ++nb) {
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t row = 8 * nb + r8;
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
          const uint32_t ch = 4 * kp + mid;  // 16-byte chunk 0..15 of the 256-byte row
          uint32_t b0, b1, b2, b3;
          gqa::ldsm_x4(sb + (ch >> 3) * C::XH + gqa::swz<128>(row, ch & 7), b0, b1, b2, b3);
          gqa::mma16816(d, ax[2 * kp], b0, b1);
          gqa::mma16816(d, ax[2 * kp + 1], b2, b3);
        }
        const int t0 = 8 * nb + 2 * c;
        s[nb][0] = (t0 < tv) ? d[0] + d[2] : -CUDART_INF_F;
        s[nb][1] = (t0 + 1 < tv) ? d[1] + d[3] : -CUDART_INF_F;
      }
      if (tv < C::TX) zero_rows(base + st * C::STAGE + 2 * C::XH, C::XH, tv, C::TX);
      softmax_pv(NbX{}, s, sb + 2 * C::XH, C::XH);
    }
    __syncwarp();
    livest[st] = next_tile(md[st], mx[st]);
    if (livest[st]) {
      if (lane == 0) fence_proxy_async();
      issue(st, md[st]);
    }
    ++j;
  }
  RK_TRACE(3, gtime());
  if (cur_u >= 0) flush(cur_u);
  RK_TRACE(4, gtime());

  RK_TRACE(5, (unsigned long long)j);
  RK_TRACE(6, (unsigned long long)nu);
  if (p.trace != nullptr && lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    RK_TRACE(7, (unsigned long long)smid);
  }
}
