// decode_ring.cuh -- the GQA decode kernel (G query heads per KV unit, 2 <= G <= 8; d = 128;
// r in {32, 64}; bf16 cache), compiled in decode_ring.cu.
//
// Alg. 2 for every unit u and query head g, with the App. C split-K online
// softmax.  Unlike decode_gqa_kernel (one private token range and ring per
// WARP), the streaming unit here is the CTA, one per SM:
//
//  * Work split.  Every unit is cut into tiles -- ceil(N/64) visual tiles of 64 tokens, then
//    ceil(M/32) text tiles of 32 full-d tokens -- and the U * tiles_per_unit tiles of the
//    batch are split into one equal contiguous range per CTA; the CTA count (decode_ring.cu,
//    ring_ctas) prefers ranges that end on unit boundaries or equal unit fractions.
//  * Producer warp (one elected thread) walks the CTA's item sequence
//        R-chunks of every unit the range touches, then the range's tiles in order
//    through a ring of NSTG (even) shared-memory stages (20 KB at r = 32: 160 KB in flight per
//    SM).  An R-chunk is 16 KB of R_r[u] rows (1-D bulk copies) plus, in a unit's first
//    chunk, q[u] (G x 128 bf16) and dmu[u]: the rotation operands are the first bytes the
//    CTA asks for, so the query rotation never queues behind the tile burst, and the tiles
//    behind them stream while the rotation runs.  Tiles are tensor-map TMA boxes (K~ [64][r]
//    with a 64/128-byte swizzle, V as two [64][64] 128-byte-swizzled halves; text K / V as
//    halves) so ldmatrix reads them without bank conflicts.
//  * Query rotation (Alg. 2 l.1-2) of the range's first unit by the eight consumer warps from
//    its R-chunk stage(s): warp w sums rows [16w, 16w + 16) of q~ = q R_r and of b = q . dmu
//    (x scale log2 e) for every head, the eight row partials are added in a fixed order
//    (deterministic) into the CTA's query table; the flusher warp rotates the other units.
//  * Eight consumer warps = two GROUPS of four; ring position p belongs to group p % 2 (NSTG
//    even: every stage has ONE consumer group, so no parity wait can be two phases behind).
//    In a tile, warp c of the group owns tokens [16c, 16c + 16) for all 128 value channels:
//    S = A . K~^T with mma.sync.m16n8k16, A rows 0..G-1 = q~ rounded to bf16 (hi), rows
//    8..8+G-1 = the remainder (lo), so q~ enters with ~16 significant bits; the online
//    softmax runs on the warp's own slice (row max over a quad, O rescaled only when a row
//    max grows), and the probabilities' C fragments ARE the A fragment of O += P . V (P hi /
//    lo rows), B from the V rows by ldmatrix.trans -- no shared-memory exchange and no
//    barrier per tile.
//  * Unit end: each warp drops its raw state (O rows hi + lo, row max, row sum) into its
//    slot and moves on; the FLUSHER warp merges the eight slots in warp order.  A unit held
//    whole is written out.  A unit shared with other CTAs is published as a partial record
//    (slot = CTA - the unit's first CTA) with an acq_rel ticket, and the LAST contributor to
//    arrive merges every record in slot order (deterministic whoever merges; no CTA ever
//    waits for another, so the launch is a plain one).  For the range's last unit the unit's
//    first CTA polls the ticket while its consumers stream and prefetches the others'
//    records; if all are in when its own state is ready it merges at once, no ticket.
//    Equal-piece plans (every unit = k <= 8 consecutive CTAs) launch one thread-block cluster
//    per unit instead: followers drop their state into their idle ring and arrive on the
//    leader's mbarrier (release.cluster); the leader's warp g reads head g of every piece
//    through distributed shared memory (ld.shared::cluster) and merges in slot order, then
//    releases the followers.  long_b16 108.4 -> 102.4 us, qwen_b8 18.3 -> 15.1, qwen_b1 18.7
//    -> 11.4 (k = 8).
//  * Variable lengths: tiles past a unit's valid length are not loaded at all (the producer
//    arrives on the stage without bytes), partially valid tiles are masked and their padded
//    V rows zeroed in shared memory before the P.V product.
//
// Measured (tools/time_decode.py, qwen_b32_r32 = 128 units x 4K tokens): with the consumers
// doing no math the launch takes 31.2 us (launch gap, first bytes, rotation, tail), with math
// 32.6 us; one CTA per unit (128 CTAs, no cross-CTA merge) beats 148 equal ranges (36.9 us:
// the unit whose middle CTA reaches it only at the END of its range waits ~4 us for that
// CTA's GPU-scope publish under the stream's load).  The per-SM stream saturates near
// 57-65 GB/s with the 8-stage ring.
//
// A stage alternating between the consumer groups lap to lap (odd NSTG, or group = tile
// parity within a unit) let a group running ahead pass a parity wait on a stage whose fill
// had not landed -- intermittent hangs / launch failures on ~225-tile ranges
// (tests/test_gpu_parity.py::test_ring_long_ranges_repeated).

template <int RK, int G>
struct RingCfg {
  static constexpr int TT = 64;                      // visual tile tokens
  static constexpr int TX = 32;                      // text tile tokens
  static constexpr int KB = TT * RK * 2;             // K~ box bytes
  static constexpr int VH = TT * 128;                // one 64-channel V half
  static constexpr int XH = TX * 128;                // one 64-channel text half
  static constexpr int STAGE = KB + 2 * VH;          // 20 KB (r = 32), 24 KB (r = 64)
  static constexpr int RROWS = 16384 / (RK * 4);     // R_r rows per chunk (16 KB)
  static constexpr int NCH = kD / RROWS;             // R chunks per unit (1 or 2)
  static constexpr int OFF_RQ = RROWS * RK * 4;      // q [G][128] bf16 in chunk 0
  static constexpr int OFF_RD = OFF_RQ + G * kD * 2; // dmu [128] f32 in chunk 0
  static constexpr int CAP = NCH == 1 ? 4 : 2;       // units per CTA range (query table)
  static constexpr int ENT = QEnt<__nv_bfloat16, RK, G>::BYTES;
  static constexpr int ULD = kD + 8;                 // unit-end slot row stride (floats): half-warp float2 stores conflict-free
  static constexpr int USLOT = 8 * G * ULD * 4;      // unit-end warp states [8 warps][G heads][ULD] f32
  static constexpr int RSCR = 8 * G * (RK + 1) * 4;  // rotation partials [8 warps][G][RK + 1]
  static constexpr int UNI = USLOT > RSCR ? USLOT : RSCR;
  static constexpr int MLCAP = 288;                  // (slot, head) pairs the flusher's merge holds
  static constexpr int PFMAX = 2;                    // partials the flusher prefetches (count - 1)
  static constexpr int OFF_TAB = 0;                  // query table [CAP] entries
  static constexpr int OFF_X = OFF_TAB + CAP * ENT;  // unit-end slots / rotation scratch (union)
  static constexpr int OFF_ML = OFF_X + UNI;         // flusher (m, l) table [MLCAP][2] f32
  static constexpr int OFF_UML = OFF_ML + MLCAP * 8; // unit-end (m, l) per warp and head [8][8][2] f32
  static constexpr int OFF_BAR = OFF_UML + 8 * 8 * 2 * 4;  // full[16] | empty[16] | rot[CAP] | rseen | ufull | ufree
  static constexpr int HDR = (OFF_BAR + (37 + CAP) * 8 + 1023) / 1024 * 1024;
  static constexpr int NSTG0 = (227 * 1024 - 1024 - HDR) / STAGE;
#ifndef RING_NSTG_CAP
#define RING_NSTG_CAP 16
#endif
  // EVEN: tiles go to the consumer groups by ring-position parity, so every stage has one
  // fixed consumer group and no waiter can fall two phases behind a stage's mbarrier (a
  // parity wait cannot tell phase k from phase k + 2; with an odd ring a stage alternated
  // between the groups and a group running ahead could pass a wait on a stale phase)
  static constexpr int NSTG = (NSTG0 < RING_NSTG_CAP ? NSTG0 : RING_NSTG_CAP) & ~1;
  static constexpr int SMEM = HDR + NSTG * STAGE + 1024;  // + alignment slack
  static constexpr int THREADS = 10 * 32;                  // producer + 8 consumers + flusher
  static_assert(STAGE % 1024 == 0 && KB % 1024 == 0, "stage alignment (swizzle atoms)");
  static_assert(OFF_RD + kD * 4 <= STAGE && 4 * XH <= STAGE, "R-chunk / text tile fit a stage");
  static_assert(NSTG >= CAP * NCH + 2, "ring must hold the R-chunks and tiles behind them");
  static_assert(NSTG % 2 == 0, "one consumer group per stage");
  static_assert(RK == 32 || RK == 64, "rank");
  static_assert(G >= 1 && G <= 8, "group");
};

struct RingMaps {
  CUtensorMap kc, v, kt, vt;
};

struct RingPlan {
  long long T;   // tiles of the batch = U * tpu
  int tpu;       // tiles per unit
  int nvt;       // visual tiles per unit
  int C;         // CTAs
  int cmax;      // partial slots per unit
  int clus;      // > 1: C = U * clus equal pieces, one cluster per unit, merged through DSMEM
  __host__ __device__ __forceinline__ long long start(int c) const { return T * c / C; }
  // CTA whose range holds tile k: the largest c with start(c) <= k
  __host__ __device__ __forceinline__ int cta_of(long long k) const { return (int)(((k + 1) * C - 1) / T); }
  // CTAs whose ranges hold tiles of unit u
  __host__ __device__ __forceinline__ int count(int u) const {
    return cta_of((long long)(u + 1) * tpu - 1) - cta_of((long long)u * tpu) + 1;
  }
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// (fence.sc.gpu, i.e. __threadfence, measured ~5 us per ticket under the decode's load)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_add_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// ---- thread-block cluster / distributed shared memory (equal-piece plans)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the shared::cluster address of this CTA's shared-memory word `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t a) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

template <int RK, int G>
__global__ void __launch_bounds__(RingCfg<RK, G>::THREADS, 1)
    decode_ring_kernel(const __grid_constant__ RingMaps maps, DecodeParams p, RingPlan pl) {
  using C = RingCfg<RK, G>;
  constexpr int NKS = RK / 16;  // score k-steps
  constexpr int S = C::NSTG;
  constexpr int kRec = kD + 4;  // partial record: acc[kD] | m | l | pad
  extern __shared__ unsigned char rsm_raw[];
  // 1024-byte aligned base (swizzle atoms), derived by pointer arithmetic on the __shared__
  // array so every access below stays a shared-memory (LDS/STS) access, not a generic one
  unsigned char* sm = rsm_raw + ((1024u - (smem_u32(rsm_raw) & 1023u)) & 1023u);
  unsigned char* ring = sm + C::HDR;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* empty = full + 16;
  uint64_t* rotb = full + 32;       // unit k >= 1 rotated (by the flusher)
  uint64_t* rseen = rotb + C::CAP;  // the consumers have seen every R-chunk land (first phase)
  uint64_t* ufull = rseen + 1;      // unit end n: the eight warps' states are in the slots (phase n)
  uint64_t* ufree = ufull + 1;      // unit end n: the flusher has read the slots (phase n)
  uint64_t* cin = ufree + 1;        // cluster leader: the other pieces' states are written
  uint64_t* cdone = cin + 1;        // cluster follower: the leader has read this CTA's state
  float* xch = reinterpret_cast<float*>(sm + C::OFF_X);  // rotation scratch (prologue)
  float* uslot = xch;                                    // unit-end warp states (after it)
  float* uml = reinterpret_cast<float*>(sm + C::OFF_UML);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = p.N, M = p.M;
  const int c_id = blockIdx.x;
  const long long kA = pl.start(c_id), kB = pl.start(c_id + 1);
  if (kA >= kB) return;
  const int uA = (int)(kA / pl.tpu), uB = (int)((kB - 1) / pl.tpu);
  const int nu = uB - uA + 1;  // <= CAP (host-checked)
  // diagnostics (rotatek_debug_decode_trace): 16 stamps per CTA
  const bool tr = p.trace != nullptr && lane == 0;
  auto stamp = [&](int slot, unsigned long long v) {
    if (tr) p.trace[(size_t)c_id * 16 + slot] = v;
  };
  if (warp == 1) stamp(0, gtime());

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);  // the four warps of the consuming group
    }
    for (int k = 0; k < C::CAP; ++k) mbar_init(&rotb[k], 1);
    mbar_init(rseen, 1);
    mbar_init(ufull, 8);
    mbar_init(ufree, 1);
    mbar_init(cin, pl.clus > 1 ? pl.clus - 1 : 1);
    mbar_init(cdone, 1);
    fence_mbar_init();
    if (pl.clus > 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (pl.clus > 1) cluster_sync_all();  // every CTA's barriers are initialised before remote arrives
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane != 0) return;
    if (p.overlap) pdl_wait();  // q is written by the preceding kernel
    tc::prefetch_tmap(&maps.kc);
    tc::prefetch_tmap(&maps.v);
    if (M > 0) {
      tc::prefetch_tmap(&maps.kt);
      tc::prefetch_tmap(&maps.vt);
    }
    const uint64_t pol = policy_evict_first();
    uint64_t pol_keep;  // rotation operands: a neighbouring CTA sharing the unit reads them too
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    int pos = 0;
    auto acquire = [&](int& s) {
      s = pos % S;
      mbar_wait(&empty[s], ((pos / S) & 1) ^ 1);
      return ring + s * C::STAGE;
    };
    for (int u = uA; u <= uB; ++u) {
      const int ur = u % p.nR;
      for (int ch = 0; ch < C::NCH; ++ch, ++pos) {
        int s;
        unsigned char* dst = acquire(s);
        const uint32_t rb = C::RROWS * RK * 4;
        const uint32_t qb = ch == 0 ? G * kD * 2 : 0, db = (ch == 0 && p.dmu) ? kD * 4 : 0;
        mbar_arrive_expect_tx(&full[s], rb + qb + db);
        bulk_g2s(dst, p.R + (size_t)ur * kD * RK + (size_t)ch * C::RROWS * RK, rb, &full[s], pol_keep);
        if (qb) bulk_g2s(dst + C::OFF_RQ, static_cast<const __nv_bfloat16*>(p.q) + (size_t)u * G * kD, qb, &full[s], pol_keep);
        if (db) bulk_g2s(dst + C::OFF_RD, p.dmu + (size_t)ur * kD, db, &full[s], pol_keep);
      }
    }
    for (int u = uA; u <= uB; ++u) {
      const long long k0 = (long long)u * pl.tpu;
      const int ja = kA > k0 ? (int)(kA - k0) : 0;
      const int jb = kB < k0 + pl.tpu ? (int)(kB - k0) : pl.tpu;
      for (int j = ja; j < jb; ++j, ++pos) {
      int s;
      unsigned char* dst = acquire(s);
      if (j < pl.nvt) {
        const int t = j * C::TT;
        const int tn = N - t < C::TT ? N - t : C::TT;
        if (valid_tn(p, u, true, t, tn) == 0) {
          mbar_arrive_cta(&full[s]);  // nothing valid: no bytes moved
          continue;
        }
        mbar_arrive_expect_tx(&full[s], C::STAGE);
        tc::tma_load_3d(dst, &maps.kc, 0, t, u, &full[s], pol);
        tc::tma_load_3d(dst + C::KB, &maps.v, 0, t, u, &full[s], pol);
        tc::tma_load_3d(dst + C::KB + C::VH, &maps.v, 64, t, u, &full[s], pol);
      } else {
        const int t = (j - pl.nvt) * C::TX;
        const int tn = M - t < C::TX ? M - t : C::TX;
        if (valid_tn(p, u, false, t, tn) == 0) {
          mbar_arrive_cta(&full[s]);
          continue;
        }
        mbar_arrive_expect_tx(&full[s], 4 * C::XH);
        tc::tma_load_3d(dst, &maps.kt, 0, t, u, &full[s], pol);
        tc::tma_load_3d(dst + C::XH, &maps.kt, 64, t, u, &full[s], pol);
        tc::tma_load_3d(dst + 2 * C::XH, &maps.vt, 0, t, u, &full[s], pol);
        tc::tma_load_3d(dst + 3 * C::XH, &maps.vt, 64, t, u, &full[s], pol);
      }
      }
    }
    return;
  }


  // ---------------- query rotation (Alg. 2 l.1-2) of unit k from its R-chunk stage(s), in one
  // fixed summation order whoever computes it: 16-row block w of q~ = q R_r as a pairwise
  // fmaf chain per lane (columns lane + 32 cc), and of b = q . dmu as a 16-lane shuffle tree;
  // the eight block partials are added in order w = 0..7
  using E = QEnt<__nv_bfloat16, RK, G>;
  auto rot_chunks = [&](int k, const unsigned char* (&chs)[C::NCH]) {
#pragma unroll
    for (int ch = 0; ch < C::NCH; ++ch) {
      const int ps = k * C::NCH + ch;  // R-chunks lead the ring: first lap
      mbar_wait(&full[ps % S], 0);
      chs[ch] = ring + (ps % S) * C::STAGE;
    }
  };
  auto rot_block = [&](int w, const unsigned char* const (&chs)[C::NCH], float (&racc)[G][RK / 32], float (&bpart)[G]) {
    const __nv_bfloat16* qs = reinterpret_cast<const __nv_bfloat16*>(chs[0] + C::OFF_RQ);
    const int i0 = 16 * w;
    const float* Rc = reinterpret_cast<const float*>(chs[i0 / C::RROWS]) + (size_t)(i0 % C::RROWS) * RK;
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int cc = 0; cc < RK / 32; ++cc) racc[gg][cc] = 0.f;
#pragma unroll
    for (int ii = 0; ii < 16; ii += 2) {
      float r0[RK / 32], r1[RK / 32];
#pragma unroll
      for (int cc = 0; cc < RK / 32; ++cc) {
        r0[cc] = Rc[ii * RK + lane + 32 * cc];
        r1[cc] = Rc[(ii + 1) * RK + lane + 32 * cc];
      }
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const float2 qv = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(qs + gg * kD + i0 + ii)[0]);
#pragma unroll
        for (int cc = 0; cc < RK / 32; ++cc) racc[gg][cc] = fmaf(qv.y, r1[cc], fmaf(qv.x, r0[cc], racc[gg][cc]));
      }
    }
    const float dmv = (p.dmu && lane < 16) ? reinterpret_cast<const float*>(chs[0] + C::OFF_RD)[i0 + lane] : 0.f;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      float v = lane < 16 ? __bfloat162float(qs[gg * kD + i0 + lane]) * dmv : 0.f;
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      bpart[gg] = v;  // lane 0
    }
  };

  // unit-end state of this CTA for head gg: the eight warp slots merged in warp order,
  // channels [4 lane, 4 lane + 4) (flusher, or the consumer warp gg for a range's last unit)
  auto own_state = [&](int gg, float4& A, float& Mx, float& Ls) {
    Mx = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < 8; ++w) Mx = fmaxf(Mx, uml[(w * 8 + gg) * 2]);
    Ls = 0.f;
    A = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const float mw = uml[(w * 8 + gg) * 2];
      const float f = (mw == -CUDART_INF_F) ? 0.f : fast_exp2(mw - Mx);
      const float4 v = reinterpret_cast<const float4*>(uslot + (w * G + gg) * C::ULD)[lane];
      Ls = fmaf(uml[(w * 8 + gg) * 2 + 1], f, Ls);
      A = make_float4(fmaf(v.x, f, A.x), fmaf(v.y, f, A.y), fmaf(v.z, f, A.z), fmaf(v.w, f, A.w));
    }
  };
  auto put = [&](int u, int gg, const float4& A, float Mx, float Ls) {  // final output or pout state
    if (p.pout) {
      float* po = p.pout + ((size_t)u * G + gg) * (kD + 2);
      po[4 * lane] = A.x; po[4 * lane + 1] = A.y; po[4 * lane + 2] = A.z; po[4 * lane + 3] = A.w;
      if (lane == 0) { po[kD] = Mx; po[kD + 1] = Ls; }
    } else {
      const float inv = 1.f / Ls;
      reinterpret_cast<float4*>(p.out + ((size_t)u * G + gg) * kD)[lane] =
          make_float4(A.x * inv, A.y * inv, A.z * inv, A.w * inv);
    }
  };
  // the range's last unit, held whole: merged by the consumer warps themselves (one head per
  // warp, in parallel) instead of the flusher
  const bool last_whole = pl.count(uB) == 1;
  // equal-piece plan with a cluster per unit: this CTA holds one piece of one unit; the pieces'
  // states are merged by the leader's consumer warps through distributed shared memory
  const bool clus_merge = pl.clus > 1;

  if (warp == 9) {
    // ------------------------------------------------------------------ flusher
    // first: the rotations of units 1.. of the range, in the background of the consumers'
    // first unit (their R-chunks landed with the first one's)
    for (int k = 1; k < nu; ++k) {
      const unsigned char* chs[C::NCH];
      rot_chunks(k, chs);
      float sum[G][RK / 32], sb[G];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        sb[gg] = 0.f;
#pragma unroll
        for (int cc = 0; cc < RK / 32; ++cc) sum[gg][cc] = 0.f;
      }
#pragma unroll 1
      for (int w = 0; w < 8; ++w) {
        float racc[G][RK / 32], bpart[G];
        rot_block(w, chs, racc, bpart);
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          sb[gg] += bpart[gg];
#pragma unroll
          for (int cc = 0; cc < RK / 32; ++cc) sum[gg][cc] += racc[gg][cc];
        }
      }
      unsigned char* ent = sm + C::OFF_TAB + k * C::ENT;
      float* qt = reinterpret_cast<float*>(ent);
      float* be = reinterpret_cast<float*>(ent + E::OFF_B);
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
#pragma unroll
        for (int cc = 0; cc < RK / 32; ++cc) qt[gg * RK + lane + 32 * cc] = sum[gg][cc] * p.sl;
        if (lane == 0) be[gg] = sb[gg] * p.sl;
      }
      const uint4* src = reinterpret_cast<const uint4*>(chs[0] + C::OFF_RQ);
      uint4* dst = reinterpret_cast<uint4*>(ent + E::OFF_Q);
      for (int e = lane; e < G * kD * 2 / 16; e += 32) dst[e] = src[e];
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cta(&rotb[k]);  // release: the table entry is written
        // the consumers wait on this chunk's first phase too; release the stage only after
        // they have (its next fill is consumed by a group that must not be two phases behind)
        mbar_wait(rseen, 0);
#pragma unroll
        for (int ch = 0; ch < C::NCH; ++ch)
          for (int a = 0; a < 4; ++a) mbar_arrive_cta(&empty[(k * C::NCH + ch) % S]);
      }
    }
    // then every unit end of the range, in unit order: the eight consumer warps' states
    // (slots, written without any barrier) are merged here in warp order while the consumers
    // stream on.  A unit held whole by this CTA is written out.  A unit shared with other CTAs
    // ("contributors", slot = CTA - the unit's first CTA) is published as a partial record
    // with a release ticket; the LAST contributor to arrive merges every slot in slot order
    // (deterministic, whoever merges) -- nobody waits for a late contributor.  Shortcut: for
    // the range's last unit, the unit's first CTA polls the ticket while its consumers stream
    // and prefetches the others' partials; if they are all in when its own state is ready it
    // merges at once with no ticket of its own (same slot-order arithmetic).
    float* ml = reinterpret_cast<float*>(sm + C::OFF_ML);
    for (int u = uA; u <= uB; ++u) {
      if (u == uB && (last_whole || clus_merge)) break;  // the consumers merge it
      const int ue = u - uA;
      const int count = pl.count(u);
      const int first = pl.cta_of((long long)u * pl.tpu);
      float* part = p.partials + (size_t)u * pl.cmax * G * kRec;
      float4 pv[C::PFMAX][G];
      float pm[C::PFMAX][G], pl_[C::PFMAX][G];
      const bool small = u == uB && count > 1 && first == c_id && count - 1 <= C::PFMAX;
      bool have = false;
      auto arrived = [&] {
        unsigned cnt = 0;
        if (lane == 0) cnt = ld_acquire_gpu(&p.counters[u]);
        return __shfl_sync(0xffffffffu, cnt, 0) == (unsigned)(count - 1);
      };
      auto prefetch = [&] {
#pragma unroll
        for (int s1 = 0; s1 < C::PFMAX; ++s1)
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            const float* src = part + ((size_t)(s1 + 1) * G + gg) * kRec;
            const bool in = s1 + 1 < count;
            pv[s1][gg] = in ? __ldcg(reinterpret_cast<const float4*>(src) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
            pm[s1][gg] = in ? __ldcg(src + kD) : -CUDART_INF_F;
            pl_[s1][gg] = in ? __ldcg(src + kD + 1) : 0.f;
          }
        have = true;
      };
      while (small && !have && !mbar_test(ufull, ue & 1)) {
        if (arrived()) prefetch();
        else __nanosleep(256);
      }
      // ---- this CTA's state of unit u, head gg: the eight warp slots merged in warp order,
      // channels [4 lane, 4 lane + 4)
      mbar_wait(ufull, ue & 1);
      if (count == 1) {
        for (int gg = 0; gg < G; ++gg) {
          float4 A; float Mx, Ls;
          own_state(gg, A, Mx, Ls);
          put(u, gg, A, Mx, Ls);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(ufree);  // the slots may take the next unit end
        continue;
      }
      if (small && (have || arrived())) {
        if (!have) prefetch();
        // every other contributor is in: merge in slot order (this CTA = slot 0), no ticket
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          float4 A; float Mx, Ls;
          own_state(gg, A, Mx, Ls);
          float M2 = Mx;
#pragma unroll
          for (int s1 = 0; s1 < C::PFMAX; ++s1) M2 = fmaxf(M2, pm[s1][gg]);
          float f = (Mx == -CUDART_INF_F) ? 0.f : fast_exp2(Mx - M2);
          float L2 = fmaf(Ls, f, 0.f);
          float4 B = make_float4(fmaf(A.x, f, 0.f), fmaf(A.y, f, 0.f), fmaf(A.z, f, 0.f), fmaf(A.w, f, 0.f));
#pragma unroll
          for (int s1 = 0; s1 < C::PFMAX; ++s1) {
            if (s1 + 1 >= count) continue;
            f = (pm[s1][gg] == -CUDART_INF_F) ? 0.f : fast_exp2(pm[s1][gg] - M2);
            L2 = fmaf(pl_[s1][gg], f, L2);
            B.x = fmaf(pv[s1][gg].x, f, B.x);
            B.y = fmaf(pv[s1][gg].y, f, B.y);
            B.z = fmaf(pv[s1][gg].z, f, B.z);
            B.w = fmaf(pv[s1][gg].w, f, B.w);
          }
          put(u, gg, B, M2, L2);
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cta(ufree);
          p.counters[u] = 0u;  // every other contributor has arrived: re-arm
        }
        stamp(15, gtime());
        continue;
      }
      // ---- publish this CTA's partial in its slot, then the release ticket
      {
        float* dst = part + (size_t)(c_id - first) * G * kRec;
        for (int gg = 0; gg < G; ++gg) {
          float4 A; float Mx, Ls;
          own_state(gg, A, Mx, Ls);
          reinterpret_cast<float4*>(dst + gg * kRec)[lane] = A;
          if (lane == 0) { dst[gg * kRec + kD] = Mx; dst[gg * kRec + kD + 1] = Ls; }
        }
      }
      __syncwarp();
      unsigned old = 0;
      if (lane == 0) {
        mbar_arrive_cta(ufree);
        // release (cumulative: the warp's partial stores, ordered before it by __syncwarp) +
        // acquire (the last arriver reads the others' partials)
        old = atom_add_acq_rel_gpu(&p.counters[u], 1u);
      }
      old = __shfl_sync(0xffffffffu, old, 0);
      if (u == uA) stamp(10, gtime());
      if (old != (unsigned)(count - 1)) continue;
      // ---- the last contributor: merge every slot in slot order
      stamp(14, gtime());
      for (int i = lane; i < count * G; i += 32) {
        ml[2 * i] = __ldcg(part + (size_t)i * kRec + kD);
        ml[2 * i + 1] = __ldcg(part + (size_t)i * kRec + kD + 1);
      }
      __syncwarp();
      for (int gg = 0; gg < G; ++gg) {
        float Mx = -CUDART_INF_F, Ls = 0.f;
        for (int s0 = 0; s0 < count; ++s0) Mx = fmaxf(Mx, ml[2 * (s0 * G + gg)]);
        float4 A = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s0 = 0; s0 < count; ++s0) {
          const int i = s0 * G + gg;
          const float ms = ml[2 * i];
          const float f = (ms == -CUDART_INF_F) ? 0.f : fast_exp2(ms - Mx);
          const float4 v = __ldcg(reinterpret_cast<const float4*>(part + (size_t)i * kRec) + lane);
          Ls = fmaf(ml[2 * i + 1], f, Ls);
          A = make_float4(fmaf(v.x, f, A.x), fmaf(v.y, f, A.y), fmaf(v.z, f, A.z), fmaf(v.w, f, A.w));
        }
        put(u, gg, A, Mx, Ls);
      }
      __syncwarp();
      if (lane == 0) p.counters[u] = 0u;  // every contributor has arrived: re-arm
    }
    stamp(4, gtime());
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int ci = warp - 1;          // 0..7
  const int grp = ci >> 2;          // tile parity this warp's group takes
  const int qd = ci & 3;            // value-channel quarter [32 qd, 32 qd + 32)
  const int ctid = threadIdx.x - 32;
  const int g = lane >> 2, c = lane & 3, mid = lane >> 3, r8 = lane & 7;
  const bool live = g < G;
  const int gl = live ? g : 0;
  const float z = live ? 1.f : 0.f;
  if (p.overlap) pdl_wait();  // out / workspace may still be read by the preceding decode

  int pos = 0;

  // ---------------- query rotation of the range's first unit (all eight warps; the flusher
  // rotates the others)
  {
    float* scr = xch;  // [8][G][RK + 1] row partials (the group exchange is not in use yet)
    const unsigned char* chs[C::NCH];
    rot_chunks(0, chs);
    // every R-chunk's first phase is observed by every consumer before the flusher releases
    // the stage (rseen), so no consumer's later parity wait on it can be two phases behind
    for (int ps = C::NCH; ps < nu * C::NCH; ++ps) mbar_wait(&full[ps], 0);
    if (warp == 1) stamp(13, gtime());
    {
      float racc[G][RK / 32], bpart[G];
      rot_block(ci, chs, racc, bpart);
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
#pragma unroll
        for (int cc = 0; cc < RK / 32; ++cc) scr[(ci * G + gg) * (RK + 1) + lane + 32 * cc] = racc[gg][cc];
        if (lane == 0) scr[(ci * G + gg) * (RK + 1) + RK] = bpart[gg];
      }
    }
    if (warp == 1) stamp(9, gtime());
    named_bar(1, 256);
    unsigned char* ent = sm + C::OFF_TAB;
    float* qt = reinterpret_cast<float*>(ent);
    float* be = reinterpret_cast<float*>(ent + E::OFF_B);
    for (int o = ctid; o < G * (RK + 1); o += 256) {
      float sum = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) sum += scr[w * G * (RK + 1) + o];
      const int gg = o / (RK + 1), jj = o % (RK + 1);
      if (jj < RK) qt[gg * RK + jj] = sum * p.sl;
      else be[gg] = sum * p.sl;
    }
    {  // raw q rows (the text keys use q)
      const uint4* src = reinterpret_cast<const uint4*>(chs[0] + C::OFF_RQ);
      uint4* dst = reinterpret_cast<uint4*>(ent + E::OFF_Q);
      for (int e = ctid; e < G * kD * 2 / 16; e += 256) dst[e] = src[e];
    }
    named_bar(1, 256);  // table entry 0 written; scratch and stage reads done
    if (grp == 0 && lane == 0)
#pragma unroll
      for (int ch = 0; ch < C::NCH; ++ch) mbar_arrive_cta(&empty[ch % S]);
    if (ci == 0 && lane == 0) mbar_arrive_cta(rseen);
    pos += nu * C::NCH;  // the other units' R-chunks are the flusher's
  }
  if (warp == 1) stamp(1, gtime());

  // per-warp running state over its token slices (all 128 value channels): rows g (q~_hi /
  // P_hi) and g + 8 (lo) of the 16 eight-channel blocks of O
  uint32_t aq[NKS][4];
  float bg = 0.f, m = -CUDART_INF_F, l = 0.f;
  float acc[16][4];
  bool first_tile = true;
  int uend = 0;  // unit ends handed to the flusher

  // this warp's 16 tokens [tb, tb + 16) of the tile: scores s[nb][.] of its two n-blocks ->
  // online softmax (row max over the quad; O rescaled only when a row max grows) -> the
  // probabilities' C fragments ARE the A fragment of O += P . V (hi / lo rows) -> 16 MMAs over
  // the 128 value channels, B from V rows [tb, tb + 16) by ldmatrix.trans
  auto softmax_pv = [&](float (&s)[2][2], uint32_t v0, uint32_t vhalf, int tb) {
    float tmax = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float mn = live ? fmaxf(m, tmax) : 0.f;
    // nothing valid yet keeps m = -inf: exp2(-inf - -inf) would be NaN
    const bool ok = live && mn != -CUDART_INF_F;
    const float alpha = (ok && mn != m) ? fast_exp2(m - mn) : 1.f;
    m = mn;
    l *= alpha;
    if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] *= alpha;
    }
    float pr[2][2];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        pr[nb][e] = ok ? fast_exp2(s[nb][e] - mn) : 0.f;
        l += pr[nb][e];
      }
    uint32_t pa[4];
    gqa::split2(pr[0][0], pr[0][1], pa[0], pa[1]);
    gqa::split2(pr[1][0], pr[1][1], pa[2], pa[3]);
    const uint32_t tok = tb + r8 + 8 * (mid & 1);
#pragma unroll
    for (int cp = 0; cp < 8; ++cp) {
      const uint32_t cb = 2 * cp + (mid >> 1);  // 8-channel block 0..15
      const uint32_t addr = v0 + (cb >> 3) * vhalf + gqa::swz<128>(tok, cb & 7);
      uint32_t b0, b1, b2, b3;
      gqa::ldsm_x4_t(addr, b0, b1, b2, b3);
      gqa::mma16816(acc[2 * cp], pa, b0, b1);
      gqa::mma16816(acc[2 * cp + 1], pa, b2, b3);
    }
  };
  // zero V rows [t0, t1) (all 128 channels, 128-byte rows in two halves) of this warp's own
  // slice: padding of variable-length units gets p = 0, but 0 * NaN would poison P.V
  auto zero_rows = [&](unsigned char* v0, int half, int t0, int t1) {
    for (int i = lane; i < (t1 - t0) * 16; i += 32) {
      const int row = t0 + i / 16, ch = i & 15;
      *reinterpret_cast<uint4*>(v0 + (ch >> 3) * half + gqa::swz<128>(row, ch & 7)) = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async();  // generic writes ordered before the stage's next TMA fill
    __syncwarp();
  };

  for (int u = uA; u <= uB; ++u) {
    if (u > uA) mbar_wait(&rotb[u - uA], 0);  // rotated by the flusher
    const unsigned char* ent = sm + C::OFF_TAB + (u - uA) * C::ENT;
    {  // per-unit state: A fragments of q~ (hi/lo rows), bias
      const float* qts = reinterpret_cast<const float*>(ent);
      const float2* t2 = reinterpret_cast<const float2*>(qts + gl * RK);
#pragma unroll
      for (int kk = 0; kk < NKS; ++kk) {
        const float2 x0 = t2[8 * kk + c], x1 = t2[8 * kk + 4 + c];
        gqa::split2(z * x0.x, z * x0.y, aq[kk][0], aq[kk][1]);
        gqa::split2(z * x1.x, z * x1.y, aq[kk][2], aq[kk][3]);
      }
      bg = z * reinterpret_cast<const float*>(ent + E::OFF_B)[gl];
      m = -CUDART_INF_F;
      l = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] = 0.f;
    }
    const long long k0 = (long long)u * pl.tpu;
    const long long ka = kA > k0 ? kA : k0, kb = kB < k0 + pl.tpu ? kB : k0 + pl.tpu;
    for (long long k = ka; k < kb; ++k, ++pos) {
      if ((pos & 1) != grp) continue;  // the stage's fixed consumer group (NSTG even)
      const int st = pos % S;
      mbar_wait(&full[st], (pos / S) & 1);
      if (warp == 1 && first_tile) stamp(2, gtime());
      if (warp == 1 && u == uA + 1 && k == ka) stamp(11, gtime());
      first_tile = false;
      unsigned char* stg = ring + st * C::STAGE;
      const uint32_t sb = smem_u32(stg);
      const int j = (int)(k - k0);
      float s[2][2];
      if (j < pl.nvt) {
        const int t = j * C::TT;
        const int tn = N - t < C::TT ? N - t : C::TT;
        const int tv = valid_tn(p, u, true, t, tn);
        const int tb = 16 * qd;  // this warp's tokens [tb, tb + 16) of the tile
        if (tv > tb) {
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            float d[4] = {0.f, 0.f, 0.f, 0.f};
            const uint32_t row = tb + 8 * nb + r8;
#pragma unroll
            for (int kp = 0; kp < RK / 32; ++kp) {
              uint32_t b0, b1, b2, b3;
              gqa::ldsm_x4(sb + gqa::swz<RK * 2>(row, 4 * kp + mid), b0, b1, b2, b3);
              gqa::mma16816(d, aq[2 * kp], b0, b1);
              gqa::mma16816(d, aq[2 * kp + 1], b2, b3);
            }
            const int t0 = tb + 8 * nb + 2 * c;
            s[nb][0] = (t0 < tv) ? d[0] + d[2] + bg : -CUDART_INF_F;
            s[nb][1] = (t0 + 1 < tv) ? d[1] + d[3] + bg : -CUDART_INF_F;
          }
          if (tv < tb + 16) zero_rows(stg + C::KB, C::VH, tv, tb + 16);
          softmax_pv(s, sb + C::KB, C::VH, tb);
        }
      } else {
        const int t = (j - pl.nvt) * C::TX;
        const int tn = M - t < C::TX ? M - t : C::TX;
        const int tv = valid_tn(p, u, false, t, tn);
        const int tb = 16 * qd;  // warps 0, 1 of the group: tokens [tb, tb + 16) of 32
        if (qd < C::TX / 16 && tv > tb) {
          // A fragments of q (x scale log2 e, hi/lo rows) from the table
          uint32_t ax[8][4];
          const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(ent + E::OFF_Q) + gl * (kD / 2);
          const float zs = z * p.sl;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const float2 lo = __bfloat1622float2(q2[8 * kk + c]), hi = __bfloat1622float2(q2[8 * kk + 4 + c]);
            gqa::split2(zs * lo.x, zs * lo.y, ax[kk][0], ax[kk][1]);
            gqa::split2(zs * hi.x, zs * hi.y, ax[kk][2], ax[kk][3]);
          }
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            float d[4] = {0.f, 0.f, 0.f, 0.f};
            const uint32_t row = tb + 8 * nb + r8;
#pragma unroll
            for (int kp = 0; kp < 4; ++kp) {
              const uint32_t chk = 4 * kp + mid;  // 16-byte chunk 0..15 of the 256-byte row
              uint32_t b0, b1, b2, b3;
              gqa::ldsm_x4(sb + (chk >> 3) * C::XH + gqa::swz<128>(row, chk & 7), b0, b1, b2, b3);
              gqa::mma16816(d, ax[2 * kp], b0, b1);
              gqa::mma16816(d, ax[2 * kp + 1], b2, b3);
            }
            const int t0 = tb + 8 * nb + 2 * c;
            s[nb][0] = (t0 < tv) ? d[0] + d[2] : -CUDART_INF_F;
            s[nb][1] = (t0 + 1 < tv) ? d[1] + d[3] : -CUDART_INF_F;
          }
          if (tv < tb + 16) zero_rows(stg + 2 * C::XH, C::XH, tv, tb + 16);
          softmax_pv(s, sb + 2 * C::XH, C::XH, tb);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[st]);
    }
    // ---------------- unit end: this warp's raw state (O rows hi + lo, row max, row sum) into
    // its slot, then on to the next unit -- the flusher merges the eight slots (no barrier)
    float lt = l + __shfl_xor_sync(0xffffffffu, l, 1);
    lt += __shfl_xor_sync(0xffffffffu, lt, 2);
    if (u == uA && (warp == 1 || warp == 5)) stamp(warp == 1 ? 8 : 12, gtime());
    if (uend > 0) mbar_wait(ufree, (uend - 1) & 1);  // the flusher has read the previous unit end
    if (live) {
      float* xrow = uslot + (ci * G + g) * C::ULD + 2 * c;
#pragma unroll
      for (int jj = 0; jj < 16; ++jj)
        *reinterpret_cast<float2*>(xrow + 8 * jj) = make_float2(acc[jj][0] + acc[jj][2], acc[jj][1] + acc[jj][3]);
      if (c == 0) {
        uml[(ci * 8 + g) * 2] = m;
        uml[(ci * 8 + g) * 2 + 1] = lt;
      }
    }
    if (u == uB && last_whole) {
      named_bar(1, 256);  // every warp's slot is written
      if (ci < G) {
        float4 A; float Mx, Ls;
        own_state(ci, A, Mx, Ls);
        put(u, ci, A, Mx, Ls);
      }
      break;
    }
    if (u == uB && clus_merge) {
      // the unit's pieces are the CTAs of this cluster (rank = slot).  A follower drops its
      // merged state, head by head, into its own (now idle) ring and signals the leader; the
      // leader's warp g reads head g of every piece through DSMEM and merges in slot order.
      named_bar(1, 256);  // every warp's slot is written
      const uint32_t rank = cluster_rank();
      float* rec = reinterpret_cast<float*>(ring);  // [G][kRec]: this piece's state
      float4 A; float Mx = -CUDART_INF_F, Ls = 0.f;
      if (ci < G) own_state(ci, A, Mx, Ls);
      if (rank != 0) {
        if (ci < G) {
          reinterpret_cast<float4*>(rec + ci * kRec)[lane] = A;
          if (lane == 0) { rec[ci * kRec + kD] = Mx; rec[ci * kRec + kD + 1] = Ls; }
        }
        named_bar(1, 256);  // the record is complete
        if (ci == 0 && lane == 0) mbar_arrive_remote(dsmem_addr(cin, 0));  // release.cluster
        if (ci == 0) mbar_wait(cdone, 0);  // stay resident until the leader has read it
      } else {
        if (ci < G) {
          mbar_wait_cluster(cin, 0);  // acquire.cluster: the other pieces' records
          float M2 = Mx;
          for (int s1 = 1; s1 < pl.clus; ++s1)
            M2 = fmaxf(M2, ld_dsmem_f32(dsmem_addr(rec + ci * kRec + kD, s1)));
          float f = (Mx == -CUDART_INF_F) ? 0.f : fast_exp2(Mx - M2);
          float L2 = fmaf(Ls, f, 0.f);
          float4 B = make_float4(fmaf(A.x, f, 0.f), fmaf(A.y, f, 0.f), fmaf(A.z, f, 0.f), fmaf(A.w, f, 0.f));
          for (int s1 = 1; s1 < pl.clus; ++s1) {
            const float ms = ld_dsmem_f32(dsmem_addr(rec + ci * kRec + kD, s1));
            const float ls = ld_dsmem_f32(dsmem_addr(rec + ci * kRec + kD + 1, s1));
            const float4 v = ld_dsmem_f4(dsmem_addr(rec + ci * kRec + 4 * lane, s1));
            f = (ms == -CUDART_INF_F) ? 0.f : fast_exp2(ms - M2);
            L2 = fmaf(ls, f, L2);
            B = make_float4(fmaf(v.x, f, B.x), fmaf(v.y, f, B.y), fmaf(v.z, f, B.z), fmaf(v.w, f, B.w));
          }
          put(u, ci, B, M2, L2);
        }
        named_bar(1, 256);  // every DSMEM read is done: release the followers
        if (ci == 0 && lane < pl.clus && lane > 0) mbar_arrive_remote(dsmem_addr(cdone, lane));
      }
      break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(ufull);
    ++uend;
  }
  if (warp == 1) {
    stamp(3, gtime());
    stamp(5, (unsigned long long)(kB - kA));
    stamp(6, (unsigned long long)nu);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    stamp(7, smid);
  }
}
