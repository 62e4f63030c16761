// decode_fast.cuh -- the streaming decode kernel (d = 128), included by decode.cu.
//
// Work decomposition: the U*(N+M) tokens of the whole batch (unit-major; within a unit
// the N visual tokens, then the M full-d text tokens) are cut into NW equal contiguous
// ranges, one per WARP.  Every warp is an independent streaming worker:
//   * lane 0 keeps STAGES tiles in flight in the warp's private shared-memory ring with
//     1-D TMA bulk copies (cp.async.bulk.shared::cluster.global.mbarrier::complete_tx,
//     SASS UBLKCP), the K~ (or K_text) tile then the V tile, both contiguous in HBM;
//   * the warp computes the tile: scores with lane groups of 32 bytes of a key row
//     (LPT lanes per token, shuffle-reduced), one online-softmax rescale per tile,
//     probabilities broadcast through shared memory, P.V with each lane owning 4 of the
//     128 value channels (two accumulator sets to halve the FMA dependency chains);
//   * tiles never straddle a unit or segment boundary; at a unit change the warp
//     flushes (m, l, acc) -- directly to `out` if it owns the whole unit, else as a
//     partial -- and the last contributor of the unit (atomic ticket) merges the
//     partials in slot order (deterministic) and re-arms the ticket.
// No CTA-level barrier exists anywhere; the CTA is only a container of WARPS warps.

template <typename T, int RK, int G, int WARPS, int STAGES, int TTV>
struct FastCfg {
  static constexpr int S = sizeof(T);
  static constexpr int CHB = 32;                       // bytes of a key row per lane
  static constexpr int CHN = CHB / S;                  // channels per lane chunk
  static constexpr int LPT_V = RK * S / CHB;           // lanes per visual token
  static constexpr int LPT_X = kD * S / CHB;           // lanes per text token
  static constexpr int TPS_V = 32 / LPT_V;             // visual tokens per step
  static constexpr int TPS_X = 32 / LPT_X;
  static constexpr int TT_V = TTV;                     // visual tile tokens
  static constexpr int STAGE = TT_V * (RK + kD) * S;   // bytes per stage
  static constexpr int XQ = (TPS_X > 4 ? TPS_X : 4);   // text tile granule (lcm(TPS_X, 4))
  static constexpr int TT_X = ((STAGE / (2 * kD * S)) / XQ) * XQ;
  static constexpr int TT_P = TT_V > TT_X ? TT_V : TT_X;
  static constexpr int VPL = kD / 32;                  // V channels per lane (4)
  static constexpr int NACC = (G == 1) ? 2 : 1;        // accumulator sets
  // per-warp shared memory
  static constexpr int OFF_Q = STAGES * STAGE;                    // float [G][kD] scaled q (G > 1)
  static constexpr int OFF_P = OFF_Q + (G > 1 ? G * kD * 4 : 0);  // float [G][TT_P] probabilities
  static constexpr int OFF_BAR = (OFF_P + G * TT_P * 4 + 7) / 8 * 8;
  static constexpr int WARP_SMEM = ((OFF_BAR + STAGES * 8) + 127) / 128 * 128;
  // CTA-shared query table: one QEnt per unit the CTA's token range touches
  static constexpr int CAP = (G == 1) ? 32 : 8;
  static constexpr int ENT = QEnt<T, RK, G>::BYTES;
  static constexpr int OFF_TAB = WARPS * WARP_SMEM;
  static constexpr int SMEM = OFF_TAB + CAP * ENT;
  static_assert(LPT_V >= 1 && LPT_V <= 32 && (32 % LPT_V) == 0, "bad RK");
  static_assert(TT_X >= XQ && TT_X % 4 == 0, "text tile too small");
  static_assert(TT_V % TPS_V == 0 && TT_V % 4 == 0, "tile");
  static_assert(STAGE % 16 == 0, "stage alignment");
};

// Warp gw's token range is [start(gw), start(gw + 1)): an equal split of the flattened
// token stream (every warp gets >= 1 token, the host guarantees >= 64).  Rounding the split
// points to the tile grid (no tensor-map box over-read at range ends, ~7 % of the GQA bytes)
// was measured no faster and is not done.
struct Split {
  long long T, L;
  int NW, N;
  __device__ __forceinline__ long long start(int gw) const { return T * gw / NW; }
  // warp whose range contains global token x
  __device__ __forceinline__ int warp_of(long long x) const {
    int g = (int)(x * NW / T);
    if (g >= NW) g = NW - 1;
    while (g + 1 < NW && start(g + 1) <= x) ++g;
    while (g > 0 && start(g) > x) --g;
    return g;
  }
};

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
  long long e;
  if (off < N) {
    tl.vis = 1; tl.t = off;
    const long long seg_end = (long long)tl.u * L + N;
    e = x + TT_V;
    if (e > seg_end) e = seg_end;
  } else {
    tl.vis = 0; tl.t = off - N;
    const long long seg_end = (long long)(tl.u + 1) * L;
    e = x + TT_X;
    if (e > seg_end) e = seg_end;
  }
  if (e > b) e = b;
  tl.tn = (int)(e - x);
  return tl;
}


__device__ __forceinline__ unsigned long long desc_pack(uint32_t end, uint32_t next) {
  return ((unsigned long long)end << 32) | next;
}

// Work-stealing tile source (decode_steal.cuh has the protocol): warp-uniform state, lane 0
// issues the atomics.  desc[w] = end << 32 | next holds warp w's unclaimed tokens.
struct StealSched {
  unsigned long long* desc;
  int gw, NW, claim, smin, lane;
  uint32_t own_x, own_e;    // owned, not yet issued: [own_x, own_e)
  unsigned long long pend;  // lane 0: result of the claim in flight
  bool pend_ok, done;

  __device__ __forceinline__ void init(bool active, long long a0, long long b0) {
    own_x = own_e = (uint32_t)a0;
    pend = 0;
    pend_ok = false;
    done = !active;
    if (!active) return;
    const uint32_t first = (uint32_t)min(a0 + claim, b0);
    if (lane == 0) {  // publish the range with the first claim taken, then claim the next
      atomicExch(&desc[gw], desc_pack((uint32_t)b0, first));
      pend = atomicAdd(&desc[gw], (unsigned long long)claim);
    }
    own_e = first;
    pend_ok = true;
  }
  // consume the claim in flight (an owner's claims are contiguous) and issue the next one
  __device__ __forceinline__ bool extend() {
    if (!pend_ok) return false;
    const unsigned long long r = __shfl_sync(0xffffffffu, pend, 0);
    pend_ok = false;
    const uint32_t nx = (uint32_t)r, en = (uint32_t)(r >> 32);
    if (nx >= en) return false;
    if (nx != own_e) own_x = nx;
    own_e = min(nx + (uint32_t)claim, en);
    if (lane == 0) pend = atomicAdd(&desc[gw], (unsigned long long)claim);
    pend_ok = true;
    return true;
  }
  // take the back half of the largest unclaimed range (>= 2 smin) and publish it as ours
  __device__ __forceinline__ bool steal() {
    for (int attempt = 0; attempt < 8; ++attempt) {
      uint32_t best = 0;
      int bv = -1;
      unsigned long long bw = 0;
      for (int v = lane; v < NW; v += 32) {
        const unsigned long long dw = *reinterpret_cast<volatile unsigned long long*>(&desc[v]);
        const uint32_t nx = (uint32_t)dw, en = (uint32_t)(dw >> 32);
        const uint32_t rem = en > nx ? en - nx : 0u;
        if (rem > best) { best = rem; bv = v; bw = dw; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const unsigned long long ow = __shfl_xor_sync(0xffffffffu, bw, o);
        if (ob > best || (ob == best && ov > bv)) { best = ob; bv = ov; bw = ow; }
      }
      if (best < 2u * (uint32_t)smin) return false;
      const uint32_t nx = (uint32_t)bw, en = (uint32_t)(bw >> 32);
      const uint32_t ne = nx + (best + 1) / 2;  // victim keeps [nx, ne), thief takes [ne, en)
      int ok = 0;
      if (lane == 0) ok = atomicCAS(&desc[bv], bw, desc_pack(ne, nx)) == bw;
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (!ok) continue;
      own_x = ne;
      own_e = min(ne + (uint32_t)claim, en);
      if (lane == 0) {
        atomicExch(&desc[gw], desc_pack(en, own_e));
        pend = atomicAdd(&desc[gw], (unsigned long long)claim);
      }
      pend_ok = true;
      return true;
    }
    return false;
  }
  // next tile (never straddles a unit/segment boundary or the owned interval)
  template <int TTV, int TTX>
  __device__ __forceinline__ bool next(Tile& tl, uint32_t& x, int N, int M) {
    if (done) return false;
    constexpr int TTM = TTV > TTX ? TTV : TTX;
    while (own_e - own_x < (uint32_t)TTM && extend()) {
    }
    if (own_x >= own_e && !steal()) {
      done = true;
      return false;
    }
    tl = tile_at<TTV, TTX>(own_x, own_e, N, M);
    x = own_x;
    own_x += tl.tn;
    return true;
  }
};

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

// Merge the `count` partial records of one unit (acc[kD] | m | l | pad per query head, slot
// order = range order, so the result is deterministic) and write out[g][:] = acc / l.
// All G heads and two slots are in flight at once: the merge is latency-bound on L2 reads
// and sits on the kernel's tail.
// pout != null (token-shard partial mode): write the merged state acc | m | l per head to
// pout [G][kD + 2] instead of the normalised output.
template <int G>
__device__ __forceinline__ void merge_unit(const float* __restrict__ part, int count,
                                           float* __restrict__ out, int lane,
                                           float* __restrict__ pout = nullptr) {
  constexpr int kRec = kD + 4;
  // pass 1 (lanes over slots): per-head max of m and the merged denominator
  // sum_s l_s 2^(m_s - max)
  float mloc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) mloc[g] = -CUDART_INF_F;
  for (int s = lane; s < count; s += 32)
#pragma unroll
    for (int g = 0; g < G; ++g) mloc[g] = fmaxf(mloc[g], __ldcg(part + ((size_t)s * G + g) * kRec + kD));
  float Ls[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    mloc[g] = warp_max(mloc[g]);
    Ls[g] = 0.f;
  }
  for (int s = lane; s < count; s += 32)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float* src = part + ((size_t)s * G + g) * kRec;
      const float ms = __ldcg(src + kD);
      const float f = (ms == -CUDART_INF_F) ? 0.f : fast_exp2(ms - mloc[g]);
      Ls[g] = fmaf(__ldcg(src + kD + 1), f, Ls[g]);
    }
#pragma unroll
  for (int g = 0; g < G; ++g) Ls[g] = warp_sum(Ls[g]);
  // pass 2 (lanes over channels): weighted sum of the accumulators; the slot weight is
  // recomputed from the (uniform) m_s load exactly as in pass 1
  float A[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) A[g][0] = A[g][1] = A[g][2] = A[g][3] = 0.f;
#pragma unroll 4
  for (int s = 0; s < count; ++s) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float* src = part + ((size_t)s * G + g) * kRec;
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src + lane * 4));
      const float ms = __ldcg(src + kD);
      const float f = (ms == -CUDART_INF_F) ? 0.f : fast_exp2(ms - mloc[g]);
      A[g][0] = fmaf(v.x, f, A[g][0]); A[g][1] = fmaf(v.y, f, A[g][1]);
      A[g][2] = fmaf(v.z, f, A[g][2]); A[g][3] = fmaf(v.w, f, A[g][3]);
    }
  }
  if (pout) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float* po = pout + (size_t)g * (kD + 2);
#pragma unroll
      for (int k = 0; k < 4; ++k) po[lane * 4 + k] = A[g][k];
      if (lane == 0) { po[kD] = mloc[g]; po[kD + 1] = Ls[g]; }
    }
    return;
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float inv = 1.f / Ls[g];
    *reinterpret_cast<float4*>(out + (size_t)g * kD + lane * 4) =
        make_float4(A[g][0] * inv, A[g][1] * inv, A[g][2] * inv, A[g][3] * inv);
  }
}

// Query rotation fused into the decode (Alg. 2 l.1-2; App. C, index reading Q14):
//   q~[g][k] = sum_i q[g][i] R_r[i][k],   b[g] = q[g] . dmu,
// pre-multiplied by scale*log2(e).  There is no separate pre-rotation launch: at kernel
// start the warps of a CTA rotate, together, every unit the CTA's token range touches into
// a CTA-shared table (rotate_cta), BEFORE any tile load is issued -- every operand (q, dmu,
// R_r rows as float4) is one independent load, so the rotation costs one round trip on an
// idle memory system.  Rotating after the first tile loads were issued queues these reads
// behind the whole-GPU tile burst (measured: +17 us/launch); one warp rotating all G = 7
// heads of its unit alone took 4 us of FMA (measured), split over the CTA it is ~4x less.
// Table entry (QEnt): qt [G][RK] f32 | b [G] f32 (16-B padded) | q [G][kD] raw dtype.
template <typename T>
__device__ __forceinline__ void unpack16(const unsigned char* p, float* f);  // 16 bytes
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const unsigned char* p, float* f) {
  const uint4 a = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) { f[2 * i] = bf16lo(w[i]); f[2 * i + 1] = bf16hi(w[i]); }
}
template <>
__device__ __forceinline__ void unpack16<float>(const unsigned char* p, float* f) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
}

// Columns [cb*CW, cb*CW + CW) of q~ (all G heads) of unit u into its table entry (one warp);
// the cb == 0 warp also stores the raw q rows and b = q . dmu.  Lane (j, r0) owns the
// float4 column block j over a contiguous block of NR rows; every operand is one
// independent load (R_r rows as float4, q rows as 16-byte chunks straight from global
// memory), so an item costs one round trip.  Splitting a unit by columns rather than by
// heads keeps each R_r byte read once per CTA (head splitting re-read it per warp and made
// G = 7 rotation 4 us, measured).
template <typename T, int RK, int CW, int G>
__device__ __forceinline__ void rotate_cols(const DecodeParams& p, int u, int cb, int lane,
                                            unsigned char* ent) {
  using E = QEnt<T, RK, G>;
  constexpr int S = sizeof(T);
  constexpr int C4 = CW / 4;                 // float4 column blocks of the item
  static_assert(C4 >= 1 && C4 <= 32 && 32 % C4 == 0 && RK % CW == 0, "columns");
  constexpr int NR = kD * C4 / 32;           // rows per lane
  constexpr int QV = 16 / S;                 // q values per 16-byte chunk
  static_assert(NR % QV == 0, "row block");
  constexpr int BATCH = NR < 32 ? NR : 32;
  const int j = lane % C4, r0 = lane / C4;
  const int ur = u % p.nR;  // nR < U: a shared (offline calibrated) rotation per kv head
  const float4* Rr = reinterpret_cast<const float4*>(p.R + (size_t)ur * kD * RK + (size_t)r0 * NR * RK +
                                                     cb * CW) + j;
  const T* qu = static_cast<const T*>(p.q) + (size_t)u * G * kD;
  float4 rv[BATCH];
#pragma unroll
  for (int t = 0; t < BATCH; ++t) rv[t] = __ldg(Rr + (size_t)t * (RK / 4));
  if (cb == 0) {
    // raw q rows into the entry (the text keys use q) and b = q . dmu
    constexpr int QCH = G * kD * S / 16;
    const uint4* qsrc = reinterpret_cast<const uint4*>(qu);
    uint4* qdst = reinterpret_cast<uint4*>(ent + E::OFF_Q);
    for (int e = lane; e < QCH; e += 32) qdst[e] = __ldg(qsrc + e);
    const float4 dm = p.dmu ? __ldg(reinterpret_cast<const float4*>(p.dmu + (size_t)ur * kD) + lane)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    float* be = reinterpret_cast<float*>(ent + E::OFF_B);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const T* qg = qu + g * kD + 4 * lane;
      float sb = Elem<T>::to_f(__ldg(qg)) * dm.x;
      sb = fmaf(Elem<T>::to_f(__ldg(qg + 1)), dm.y, sb);
      sb = fmaf(Elem<T>::to_f(__ldg(qg + 2)), dm.z, sb);
      sb = fmaf(Elem<T>::to_f(__ldg(qg + 3)), dm.w, sb);
      sb = warp_sum(sb);
      if (lane == 0) be[g] = sb * p.sl;
    }
  }
  float acc[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
#pragma unroll
  for (int s0 = 0; s0 < NR; s0 += BATCH) {
    if (s0 > 0) {
#pragma unroll
      for (int t = 0; t < BATCH; ++t) rv[t] = __ldg(Rr + (size_t)(s0 + t) * (RK / 4));
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint4* qrow = reinterpret_cast<const uint4*>(qu + g * kD + r0 * NR + s0);
#pragma unroll
      for (int v = 0; v < BATCH / QV; ++v) {
        const uint4 qc = __ldg(qrow + v);
        float qf[QV];
        unpack16<T>(reinterpret_cast<const unsigned char*>(&qc), qf);
#pragma unroll
        for (int e = 0; e < QV; ++e) {
          const float4 r4 = rv[v * QV + e];
          acc[g][0] = fmaf(qf[e], r4.x, acc[g][0]);
          acc[g][1] = fmaf(qf[e], r4.y, acc[g][1]);
          acc[g][2] = fmaf(qf[e], r4.z, acc[g][2]);
          acc[g][3] = fmaf(qf[e], r4.w, acc[g][3]);
        }
      }
    }
  }
#pragma unroll
  for (int o = C4; o < 32; o <<= 1)
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[g][k] += __shfl_xor_sync(0xffffffffu, acc[g][k], o);
  if (lane < C4) {
    float* qt = reinterpret_cast<float*>(ent);
#pragma unroll
    for (int g = 0; g < G; ++g)
      *reinterpret_cast<float4*>(qt + g * RK + cb * CW + 4 * j) =
          make_float4(acc[g][0] * p.sl, acc[g][1] * p.sl, acc[g][2] * p.sl, acc[g][3] * p.sl);
  }
}

// CTA-cooperative rotation of the nu units [uA, uA + nu) the CTA's range touches: work
// items are (unit, column block); the split PU (columns per item = RK / PU) is the largest
// power of two with nu * PU <= warps, so the CTA's warps get ~one item each.
template <typename T, int RK, int G, int PU, int ENT>
__device__ __forceinline__ void rotate_items(const DecodeParams& p, int uA, int nu, int w, int nw,
                                             int lane, unsigned char* tab) {
  for (int it = w; it < nu * PU; it += nw)
    rotate_cols<T, RK, RK / PU, G>(p, uA + it / PU, it % PU, lane, tab + (it / PU) * ENT);
}

// Runs before any tile load is issued: issuing the first tiles before (or right after) the
// rotation's reads was measured 1-2 us slower -- the reads queue behind the tile burst.
template <typename T, int RK, int G, int WARPS, int ENT>
__device__ __forceinline__ void rotate_cta(const DecodeParams& p, int uA, int nu, int w, int lane,
                                           unsigned char* tab) {
  constexpr int S = sizeof(T);
  // ROTATEK_DECODE_OVERLAP: q (and the workspace) may still be in flight from the preceding
  // kernel; every thread waits for it here (the first tile loads are already issued)
  if (p.overlap) pdl_wait();
  int pu = 1;
  while (2 * pu * nu <= WARPS && 2 * pu <= 8) pu *= 2;
  // columns per item must keep >= one 16-byte q chunk of rows per lane: CW >= 4 * (16/S) / (kD/32)
  constexpr int CWMIN = (16 / S) * 4 * 32 / kD;
  if (pu >= 8 && RK / 8 >= CWMIN)
    rotate_items<T, RK, G, (RK / 8 >= CWMIN ? 8 : 1), ENT>(p, uA, nu, w, WARPS, lane, tab);
  else if (pu >= 4 && RK / 4 >= CWMIN)
    rotate_items<T, RK, G, (RK / 4 >= CWMIN ? 4 : 1), ENT>(p, uA, nu, w, WARPS, lane, tab);
  else if (pu >= 2 && RK / 2 >= CWMIN)
    rotate_items<T, RK, G, (RK / 2 >= CWMIN ? 2 : 1), ENT>(p, uA, nu, w, WARPS, lane, tab);
  else
    rotate_items<T, RK, G, 1, ENT>(p, uA, nu, w, WARPS, lane, tab);
  __syncthreads();
}

// the CTA's token range [ca, cb) (union of its warps' ranges) and the units it touches
__device__ __forceinline__ void cta_units(const Split& sp, int WARPS, int blk, int& uA, int& nu) {
  const int NW = sp.NW;
  const long long L = sp.L;
  const int w0 = blk * WARPS, w1 = (blk + 1) * WARPS < NW ? (blk + 1) * WARPS : NW;
  const long long ca = sp.start(w0), cb = sp.start(w1);
  uA = (int)(ca / L);
  nu = cb > ca ? (int)((cb - 1) / L) - uA + 1 : 0;
}

// One tile: scores (key rows of KR channels), online-softmax rescale, P.V.
// FULL: tn == TT (branch-free, fully unrolled); else the tail path.
template <typename T, int KR, int TT, int G, int NACC, bool FULL, bool BIAS>
__device__ __forceinline__ void tile_compute(const unsigned char* __restrict__ kbuf,
                                             const unsigned char* __restrict__ vbuf, int tn,
                                             const float* __restrict__ qsm,
                                             const float (&qreg)[32 / sizeof(T)],
                                             const float* __restrict__ bs, float* __restrict__ pbuf,
                                             float (&m)[G], float (&l)[G],
                                             float (&acc)[NACC][G][4], int lane) {
  constexpr int S = sizeof(T);
  constexpr int CHN = 32 / S;
  constexpr int LPT = KR * S / 32;
  constexpr int TPS = 32 / LPT;
  constexpr int NS = TT / TPS;
  const int cv = lane % LPT, tv = lane / LPT;
  float sc[G][NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int tok = s * TPS + tv;
    float kf[CHN];
    unpack_chunk<T>(kbuf + (size_t)tok * KR * S + cv * 32, kf);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float d0 = 0.f, d1 = 0.f;
      if constexpr (G == 1) {
#pragma unroll
        for (int i = 0; i < CHN; i += 2) {
          d0 = fmaf(qreg[i], kf[i], d0);
          d1 = fmaf(qreg[i + 1], kf[i + 1], d1);
        }
      } else {
        const float* qq = qsm + g * KR + cv * CHN;
#pragma unroll
        for (int i = 0; i < CHN; i += 4) {
          const float4 q4 = *reinterpret_cast<const float4*>(qq + i);
          d0 = fmaf(q4.x, kf[i], d0);
          d1 = fmaf(q4.y, kf[i + 1], d1);
          d0 = fmaf(q4.z, kf[i + 2], d0);
          d1 = fmaf(q4.w, kf[i + 3], d1);
        }
      }
      float dsum = d0 + d1;
#pragma unroll
      for (int o = 1; o < LPT; o <<= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
      if constexpr (BIAS) dsum += bs[g];
      sc[g][s] = (FULL || tok < tn) ? dsum : -CUDART_INF_F;
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float tmax = sc[g][0];
#pragma unroll
    for (int s = 1; s < NS; ++s) tmax = fmaxf(tmax, sc[g][s]);
#pragma unroll
    for (int o = 16; o >= LPT; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    const float mn = fmaxf(m[g], tmax);
    const float alpha = fast_exp2(m[g] - mn);
    m[g] = mn;
    l[g] *= alpha;
#pragma unroll
    for (int a = 0; a < NACC; ++a)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[a][g][k] *= alpha;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float pr = fast_exp2(sc[g][s] - mn);
      if (cv == 0) {
        l[g] += pr;
        pbuf[g * TT + s * TPS + tv] = pr;
      }
    }
  }
  __syncwarp();
  if constexpr (FULL) {
#pragma unroll
    for (int t4 = 0; t4 < TT / 4; ++t4) {
      float4 pg[G];
#pragma unroll
      for (int g = 0; g < G; ++g) pg[g] = *reinterpret_cast<const float4*>(pbuf + g * TT + 4 * t4);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float vf[4];
        load_v4<T>(vbuf + (size_t)(4 * t4 + j) * kD * S + lane * 4 * S, vf);
        const int a = j % NACC;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float pj = j == 0 ? pg[g].x : j == 1 ? pg[g].y : j == 2 ? pg[g].z : pg[g].w;
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[a][g][k] = fmaf(pj, vf[k], acc[a][g][k]);
        }
      }
    }
  } else {
    for (int t = 0; t < tn; ++t) {
      float vf[4];
      load_v4<T>(vbuf + (size_t)t * kD * S + lane * 4 * S, vf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pj = pbuf[g * TT + t];
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[0][g][k] = fmaf(pj, vf[k], acc[0][g][k]);
      }
    }
  }
  __syncwarp();
}

template <typename T, int RK, int G, int WARPS, int STAGES, int TTV, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) decode_fast_kernel(DecodeParams p, int NW, int cmax) {
  using C = FastCfg<T, RK, G, WARPS, STAGES, TTV>;
  constexpr int NACC = C::NACC;
  extern __shared__ __align__(128) unsigned char fsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * p.aw + w;
  unsigned char* base = fsm + w * C::WARP_SMEM;
  float* qs = reinterpret_cast<float*>(base + C::OFF_Q);
  float* pbuf = reinterpret_cast<float*>(base + C::OFF_P);
  unsigned char* tab = fsm + C::OFF_TAB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::OFF_BAR);

  const int N = p.N, M = p.M;
  const long long L = (long long)N + M;
  const long long Ttot = L * p.U;
  RK_TRACE(0, gtime());
  int uA, nu;
  const Split sp{Ttot, L, NW, N};
  cta_units(sp, p.aw, blockIdx.x, uA, nu);
  const long long a = sp.start(gw), b = sp.start(gw + 1);
  const bool active = w < p.aw && gw < NW && a < b;

  const T* Kc = static_cast<const T*>(p.Kc);
  const T* V = static_cast<const T*>(p.V);
  const T* Kt = static_cast<const T*>(p.Kt);
  const T* Vt = static_cast<const T*>(p.Vt);
  const uint64_t pol = policy_evict_first();

  if (active && lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  // ---------------- producer (lane 0): issue the tile at cursor px into stage st
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
      bulk_g2s(dst, Kt + ((size_t)tl.u * p.Ms + tl.t) * kD, kb, &bar[st], pol);
      bulk_g2s(dst + C::TT_X * kD * C::S, Vt + ((size_t)tl.u * p.Ms + tl.t) * kD, kb, &bar[st], pol);
    }
    px += tl.tn;
  };
  pdl_launch_dependents();
  // query table, then tiles -- or, when launched overlapped with the preceding kernel, the
  // first tiles (cache bytes are complete by contract) while it finishes, then the table
  if (p.overlap && active && lane == 0)
    for (int s = 0; s < STAGES && px < b; ++s) issue(s);
  rotate_cta<T, RK, G, WARPS, C::ENT>(p, uA, nu, w, lane, tab);
  RK_TRACE(1, gtime());
  if (!active) return;
  if (!p.overlap && lane == 0)
    for (int s = 0; s < STAGES && px < b; ++s) issue(s);

  // ---------------- consumer state
  float m[G], l[G], acc[NACC][G][4];
  float qreg[C::CHN], xreg[C::CHN];  // register copies of q~ / q chunks when G == 1
  int cur_u = -1;

  const float* qts = nullptr;  // current unit's scaled q~ [G][RK] and bias [G] (table entry)
  const float* bs = nullptr;
  auto setup = [&](int u) {
    const unsigned char* ent = tab + (u - uA) * C::ENT;
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

  // the last arrival at a unit's ticket merges its partials (deferring the first unit's
  // arrival to the end of the range was measured slower: it serialises two merges in the
  // tail)
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
    const long long x0 = (long long)u * L, x1 = x0 + L - 1;
    const int first = sp.warp_of(x0), last = sp.warp_of(x1);
    const int count = last - first + 1;
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
    if (count == 1 && p.pout) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float* po = p.pout + ((size_t)u * G + g) * (kD + 2);
#pragma unroll
        for (int k = 0; k < 4; ++k) po[lane * 4 + k] = A[g][k];
        if (lane == 0) { po[kD] = m[g]; po[kD + 1] = lt[g]; }
      }
      return;
    }
    if (count == 1) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float inv = 1.f / lt[g];
        *reinterpret_cast<float4*>(p.out + ((size_t)u * G + g) * kD + lane * 4) =
            make_float4(A[g][0] * inv, A[g][1] * inv, A[g][2] * inv, A[g][3] * inv);
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
      *reinterpret_cast<float4*>(dst + lane * 4) = make_float4(A[g][0], A[g][1], A[g][2], A[g][3]);
    }
    arrive(u, count);
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
    // refill this stage with the tile STAGES ahead (the whole warp has consumed it)
    if (lane == 0 && px < b) {
      fence_proxy_async();
      issue(st);
    }
    cx += tl.tn;
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
