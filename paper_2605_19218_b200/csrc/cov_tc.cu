// cov_tc.cu -- Alg. 1 lines 1-3: the key Gram matrix S = sum_n K_n K_n^T and the
// column sums sum_n K_n, on the 5th-generation tensor cores (tcgen05) for d = 128, bf16 keys.
//
//   C = K^T K as one GEMM D[d x d] = A[d x tok] . B[tok x d] where A = K^T and B = K are the
//   SAME shared-memory tile read through two MN-major descriptors (128-byte swizzle).
//   TMA (cp.async.bulk.tensor.3d, SWIZZLE_128B) brings 128-token x 128-channel chunks into a
//   4-stage ring; one elected thread issues 8 tcgen05.mma (M=128, N=144, K=16) per chunk into
//   one of two fp32 accumulators in TMEM.  N = 144: B = [K | 1] -- every ring stage holds a
//   third 64-element atom of bf16 ones (written once, never touched by TMA), so accumulator
//   columns 128..143 are the column sums sum_n K[n][i] (no separate MMA, no shared-memory
//   pass).  Sixteen epilogue warps drain the other accumulator with tcgen05.ld and add it into
//   fp64 registers, so each fp32 accumulation spans at most 256 tokens (exact bf16 products,
//   fp32 per window, fp64 across windows: the precision scheme of SURVEY Appendix A E-5/E-6).  PERSISTENT: one CTA per SM walks its (unit,
//   part) items with running stage / window counters, so the next item's loads and MMAs
//   overlap this item's epilogue.  Out-of-range tokens are zero-filled by TMA.
//   llava_b32 (ncu): 290 us (one CTA per unit) -> 214 -> 229 (r1 final) -> 218 (16 epilogue
//   warps of 32 columns, TMEM released as soon as a window is in registers, no divisions in
//   the finalize) -> 191 (column sums folded into the Gram MMA instead of 8 extra N = 16 MMAs
//   per chunk) -> 178 (only the 10 blocks on/above the diagonal drained, mirrored writes)
//   -> 165 (every block drained again, all written transposed: coalesced stores, see the
//   epilogue) -> 160 (per-column finalize factors staged in shared memory once per unit:
//   0.80 of the copy peak); 512-token windows 167 us but less precise (see kWin).  (fp32 TwoSum
//   pairs instead of F2F.F64.F32 + DADD in the drain: 203 us, register spills -- not kept.)
//
// Warp roles (576 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2..17 epilogue (TMEM lane quadrant = warp % 4, column quarter = (warp - 2) / 4).
#include <cstdio>
#include <cstring>

#include "internal.h"
#include "tc_common.cuh"
#include "tok_gather.cuh"

namespace rk {

namespace {
constexpr int kTK = 128;                 // tokens per chunk (fp32 accumulation window)
constexpr int kDc = 128;                 // head dim
#ifndef COV_STAGES
#define COV_STAGES 4
#endif
#ifdef COV_DIAG_NOFIN
constexpr bool kDiagNoFin = true;  // diagnostics build only: no finalize / partial writes
#else
constexpr bool kDiagNoFin = false;
#endif
// 2, 3 and 4 stages measured equal (r2, tools/run_covdiag.sh); 6 slower (254 vs 229 us)
constexpr int kStages = COV_STAGES;
// chunks per fp32 TMEM accumulation window: 256 tokens (SURVEY E-6).  512 was measured (r2,
// tools/cov_err2.py): 191 -> 167 us on llava_b32 (half the fp32 -> fp64 drains), but the worst
// unit's projector error vs the fp64 oracle on large-mean planted-gap keys grows 9.7e-5 ->
// 1.4e-4 (40 units x 300 tokens; the CUDA-core path: 2.5e-6), past the 1e-4 gate -- not taken
constexpr int kWin = 2;
constexpr int kHalfBytes = kTK * 128;    // one 64-channel half: kTK rows x 128 B
// a stage = the chunk's two 64-channel halves + a third "half" of bf16 ones: the Gram MMA runs
// with N = 144 (B = [K | 1]), so its columns 128..143 are the column sums sum_n K[n][i]
constexpr int kStageBytes = 3 * kHalfBytes;
constexpr int kEpiWarps = 16;               // 4 per TMEM lane quadrant, 32 accumulator columns each
constexpr int kThreads = (2 + kEpiWarps) * 32;
constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
constexpr int kAcc = 2;                    // TMEM accumulators (3 measured: no change; a = gw & 1)
constexpr int kAccCols = 256;              // TMEM columns per accumulation window (144 used)
constexpr int kTmemCols = 512;             // kAcc windows x kAccCols (128 Gram + 16 column-sum columns used)
}  // namespace

__global__ void __launch_bounds__(kThreads, 1) cov_tc_kernel(const __grid_constant__ CUtensorMap tmap, int N,
                                                             int U, int parts, double* __restrict__ covpart,
                                                             double* __restrict__ colpart,
                                                             const double* __restrict__ sigma,
                                                             double* __restrict__ cq, double* __restrict__ mu,
                                                             bool center, bool fused, TokSrc tsrc,
                                                             const __nv_bfloat16* __restrict__ Kg) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + kAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAcc);
  __shared__ double colsum_sm[kDc];
  __shared__ double2 fac_sm[kDc];  // fused finalize: (s_c, s_c mu_c n) per column

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PERSISTENT: this CTA takes the work items (u, p) = blockIdx.x, + gridDim.x, ...; the ring
  // stages and the two TMEM accumulators run continuously across items (running chunk and
  // window counters), so the next item's loads and MMAs overlap this item's epilogue
  const int nchunks_all = (N + kTK - 1) / kTK;
  const int nitems = U * parts;
  auto item_range = [&](int it, int& u, int& p, int& c_lo, int& nch) {
    u = it / parts;
    p = it % parts;
    c_lo = (int)((long long)nchunks_all * p / parts);
    nch = (int)((long long)nchunks_all * (p + 1) / parts) - c_lo;
  };

  const bool gathered = tsrc.active();  // token list / per-unit lengths: cp.async producer
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], gathered ? 32 : 1);
      mbar_init(&empty[s], 1);  // released by the MMA commit alone (no smem column-sum pass)
    }
    for (int a = 0; a < kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    fence_mbar_init();
    tc::prefetch_tmap(&tmap);
  }
  // column sums on the tensor core too: every stage's third half is all ones (never written by
  // TMA), so D[:, 128 + j] = K^T . ONES = sum_n K[n][i] (all 16 columns equal)
  for (int st = 0; st < kStages; ++st)
    for (int e = threadIdx.x; e < kHalfBytes / 16; e += blockDim.x)
      reinterpret_cast<uint4*>(sm + st * kStageBytes + 2 * kHalfBytes)[e] =
          make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  fence_proxy_async();  // generic-proxy writes must be visible to the tensor core (async proxy)
  if (warp == 1) tc::tmem_alloc(tmem_slot, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && gathered) {
    // all 32 lanes gather the chunk's rows (tok_gather.cuh); zero rows past the unit's count
    int gi = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      int u, p, c_lo, nch;
      item_range(it, u, p, c_lo, nch);
      const int nv = tsrc.valid(u, N);
      for (int i = 0; i < nch; ++i, ++gi) {
        const int s = gi % kStages;
        mbar_wait(&empty[s], ((gi / kStages) & 1) ^ 1);
        gather_tile_128x128(tsrc, Kg, u, N, nv, (c_lo + i) * kTK, sm + s * kStageBytes, kHalfBytes, lane);
        cp_async_arrive_noinc(&full[s]);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int gi = 0;  // running chunk counter (ring stage / phase)
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        int u, p, c_lo, nch;
        item_range(it, u, p, c_lo, nch);
        for (int i = 0; i < nch; ++i, ++gi) {
          const int s = gi % kStages;
          mbar_wait(&empty[s], ((gi / kStages) & 1) ^ 1);
          unsigned char* dst = sm + s * kStageBytes;
          mbar_arrive_expect_tx(&full[s], 2 * kHalfBytes);
          const int tok = (c_lo + i) * kTK;
          tc::tma_load_3d(dst, &tmap, 0, tok, u, &full[s], pol);
          tc::tma_load_3d(dst + kHalfBytes, &tmap, 64, tok, u, &full[s], pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, 144, true, true);  // B = [K | 1]
      int gi = 0, gw = 0;  // running chunk / accumulation-window counters
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        int u, p, c_lo, nch;
        item_range(it, u, p, c_lo, nch);
        (void)u; (void)p; (void)c_lo;
        for (int i = 0; i < nch; ++i, ++gi) {
          // fp32 accumulation window = kWin chunks (kWin * 128 = 256 tokens, E-6), never
          // spanning two items
          const int s = gi % kStages, a = gw & 1;
          const bool first = (i % kWin) == 0, last = (i % kWin) == kWin - 1 || i == nch - 1;
          mbar_wait(&full[s], (gi / kStages) & 1);
          if (gathered) fence_proxy_async();  // cp.async (generic proxy) writes -> tensor core
          if (first) mbar_wait(&tempty[a], ((gw >> 1) & 1) ^ 1);
          tc::fence_after();
          const uint32_t base = smem_u32(sm + s * kStageBytes);
#pragma unroll
          for (int kk = 0; kk < kTK / 16; ++kk) {
            // MN-major, SWIZZLE_128B: LBO = next 64-channel half, SBO = next 8-token group
            const uint64_t desc = tc::smem_desc(base + kk * 16 * 128, kHalfBytes, 1024, tc::SWZ_128B);
#ifndef COV_DIAG_NOMMA  // diagnostics build only: stream without the Gram MMAs
            tc::mma_bf16(tmem + a * kAccCols, desc, desc, idesc, (first && kk == 0) ? 0u : 1u);
#else
            (void)desc;
#endif
          }
          tc::commit(&empty[s]);
          if (last) {
            tc::commit(&tfull[a]);
            ++gw;
          }
        }
      }
    }
  } else {
    // ---------------- epilogue: 16 warps (warp w reads TMEM lane quadrant w % 4; the four
    // warps of a quadrant take 32 accumulator columns each)
    const int e = warp - 2;
    const int q = warp & 3;        // TMEM lane quadrant this warp may access
    const int h = e >> 2;          // accumulator column quarter
    const int row = 32 * q + lane;  // output row (channel i)
    // Output: each warp writes its 32 x 32 block TRANSPOSED -- lane = row i of the block,
    // stores go to C[32h + j][32q + lane], so every store instruction covers 32 consecutive
    // doubles (256 B).  S = K^T K is symmetric (D[i][j] and D[j][i] are the same products
    // summed in the same order), so the transposed block is block (h, q) of S, and every
    // block is written exactly once.  Row-major stores from this layout put the lanes 1 KB
    // apart (32 sectors per instruction): 178 -> 165 us on llava_b32 (ncu).  Measured and not
    // kept (tools/run_covdiag*.sh): draining only the 10 blocks on/above the diagonal with the
    // other 6 written from a shared-memory staging (166 us); 2 or 3 ring stages (equal); a
    // third TMEM accumulator (equal).  The ablations put the rest above the pure TMA stream
    // (111 us, 6.8 TB/s) into the fp64 drain and the per-unit finalize.
    const int et = e * 32 + lane;   // 0..511
    constexpr int kEpiThreads = kEpiWarps * 32;
    int gi = 0, gw = 0;  // running chunk / window counters (as the producer and MMA warps)
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    int u, p, c_lo, nch;
    item_range(it, u, p, c_lo, nch);
    (void)c_lo;
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    double csum = 0.0;  // column sum of channel `row` (warps of column quarter 0)
    for (int i = 0; i < nch; ++i, ++gi) {
      const int a = gw & 1, wph = (gw >> 1) & 1;
      const bool last = (i % kWin) == kWin - 1 || i == nch - 1;
      if (!last) continue;
      // drain the window's accumulator into fp64 (both loads in flight, one wait)
      mbar_wait(&tfull[a], wph);
      ++gw;
      tc::fence_after();
      const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16) + a * kAccCols;
      uint32_t r[2][16], rc = 0;
      if (h == 0) tc::ld_32x32b_x1(tq + 128, rc);
#pragma unroll
      for (int b = 0; b < 2; ++b) tc::ld_32x32b_x16(tq + h * 32 + b * 16, r[b]);
      tc::ld_wait();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[a]);  // the registers hold the window: free TMEM
#ifndef COV_DIAG_NODRAIN  // diagnostics build only: skip the fp64 accumulation
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[b * 16 + j] += (double)__uint_as_float(r[b][j]);
#else
      acc[0] += (double)__uint_as_float(r[0][0] ^ r[1][15]);
#endif
      if (h == 0) csum += (double)__uint_as_float(rc);
    }
    if (h == 0) colsum_sm[row] = csum;
    asm volatile("bar.sync 1, %0;" ::"r"(kEpiThreads) : "memory");
    if (fused && !kDiagNoFin) {
      // parts == 1: this CTA saw every token of the unit -> finalize here (mu, C, C_q):
      //   C_q[r][c] = s_r s_c (S_rc - n mu_r mu_c) = (s_r s_c) S_rc - (s_r mu_r)(s_c mu_c n)
      // with the per-column factors (s_c, s_c mu_c n) staged in shared memory once per unit
      const double nu = (double)tsrc.valid(u, N);  // tokens of the unit (per-unit lengths)
      const double inv_nu = 1.0 / nu;
      if (et < kDc) {
        const double m = center ? colsum_sm[et] * inv_nu : 0.0;
        const double sgc = sigma[(size_t)u * kDc + et];
        fac_sm[et] = make_double2(sgc, sgc * m * nu);
        mu[(size_t)u * kDc + et] = center ? colsum_sm[et] / nu : 0.0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kEpiThreads) : "memory");
      const double2 fr = fac_sm[row];
      const double sr = fr.x, srm = fr.y * inv_nu;  // s_r, s_r mu_r
      double* cqt = cq + (size_t)u * kDc * kDc + (size_t)(h * 32) * kDc + row;  // column `row`
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double2 fc = fac_sm[h * 32 + j];
        cqt[(size_t)j * kDc] = fma(sr * fc.x, acc[j], -srm * fc.y);
      }
    } else if (!kDiagNoFin) {
      double* outt = covpart + ((size_t)u * parts + p) * kDc * kDc + (size_t)(h * 32) * kDc + row;
#pragma unroll
      for (int j = 0; j < 32; ++j) outt[(size_t)j * kDc] = acc[j];
      if (et < kDc) colpart[((size_t)u * parts + p) * kDc + et] = colsum_sm[et];
    }
    // every epilogue warp is done reading colsum_sm before the next item's drain may
    // overwrite it (write-after-read across items of this persistent CTA)
    asm volatile("bar.sync 1, %0;" ::"r"(kEpiThreads) : "memory");
  }
    }  // items
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, kTmemCols);
  }
}

// ------------------------------------------------------------------------------ host
using PFN_encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encode get_encode() {
  static PFN_encode fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_encode>(p);
  }();
  return fn;
}

bool encode_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                         uint32_t b1, int swizzle_bytes) {
  return encode_tmap_3d_bf16_strided(map, base, d0, d1, d2, d1, b0, b1, swizzle_bytes);
}

bool encode_tmap_3d_bf16_strided(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                                 uint64_t d1_stride, uint32_t b0, uint32_t b1, int swizzle_bytes) {
  PFN_encode enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1_stride * 2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool cov_tc_supported(int d, bool bf16) { return bf16 && d == kDc && get_encode() != nullptr; }

int launch_cov_tc(int U, int N, bool center, const void* K, const CalibWs& ws, cudaStream_t st,
                  bool allow_fused, const TokSrc& tsrc) {
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  if (!tsrc.active() && !encode_tmap_3d_bf16(&map, K, kDc, (uint64_t)N, (uint64_t)U, 64, kTK, 128)) return -2;
  static int attr_slot[kMaxDevices];
  once_per_device(attr_slot, [] {
    cudaFuncSetAttribute(cov_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    return 1;
  });
  // persistent: one CTA per SM over the U * parts work items (the ring runs across items)
  const int nitems = U * ws.parts;
  const int grid = nitems < kNumSMs ? nitems : kNumSMs;
  // parts == 1: the kernel also finalizes (mu, C = S - N mu mu^T, C_q) -- no finalize launch
  cov_tc_kernel<<<grid, kThreads, kSmem, st>>>(map, N, U, ws.parts, ws.covpart, ws.colpart, ws.sigma, ws.cq,
                                               ws.mu, center, allow_fused && ws.parts == 1, tsrc,
                                               static_cast<const __nv_bfloat16*>(K));
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rk
