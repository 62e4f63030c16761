// compress_tc.cu -- Alg. 1 line 14, K~ = RNE(K R_r), on tcgen05 for d = 128, bf16.
//
// D[128 tokens x r] = A[128 tokens x 128 channels] . B[128 channels x r] per tile:
//   * A (K-major, SWIZZLE_128B) is the key tile brought by TMA (two 64-channel halves);
//   * B is R_r split EXACTLY into three bf16 matrices, R = hi + mid + lo (8 + 8 + 8 significant
//     bits cover fp32's 24), written once per CTA into shared memory as K-major swizzled R^T;
//   * 3 x 8 tcgen05.mma (M=128, N=r, K=16) accumulate K.hi + K.mid + K.lo into one fp32 TMEM
//     accumulator (bf16 x bf16 products are exact), so K~ matches an fp32 GEMM with the stored
//     fp32 R -- the same R the decode uses for q~ (reading R-store in DESIGN.md);
//   * four epilogue warps read the accumulator (tcgen05.ld), round to bf16 (RNE) and store
//     their token rows (a warp writes 32 consecutive rows: one contiguous block).
// Work item = (unit, token part); a CTA streams its part through a 3-stage TMA ring with
// double-buffered TMEM accumulators.  Tokens past N are zero-filled by TMA and not stored.
#include <cstdio>
#include <cstring>

#include "internal.h"
#include "tc_common.cuh"

namespace rk {

namespace {
constexpr int kTM = 128;                      // tokens per tile (MMA M)
constexpr int kDc = 128;
constexpr int kStages = 2;                    // 2 x 32 KB: two CTAs per SM (one's prologue /
                                              // epilogue overlaps the other's stream; 3 stages
                                              // with one CTA per SM: 214 vs 175 us, llava_b32)
constexpr int kHalf = kTM * 128;              // one 64-channel half of a key tile
constexpr int kStageBytes = 2 * kHalf;        // 32 KB
constexpr int kThreads = 192;                 // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
}  // namespace

template <int RK>
struct CmpCfg {
  static constexpr int B_HALF = RK * 128;                  // r rows x 64 channels x 2 B
  static constexpr int B_SPLIT = 2 * B_HALF;                // both channel halves
  static constexpr int B_BYTES = 3 * B_SPLIT;               // hi, mid, lo
  static constexpr int TMEM_COLS = (2 * RK <= 32) ? 32 : (2 * RK <= 64) ? 64 : (2 * RK <= 128) ? 128 : 256;
  // r <= 32: the epilogue stages each warp's 32 output rows (32 x r bf16) in shared memory and
  // writes them as one contiguous block (r = 64 / 128 would not fit two CTAs per SM)
  static constexpr bool STAGE_OUT = RK <= 32;
  static constexpr int CPR = RK / 8;                       // 16-byte chunks per output row
  static constexpr int OUT_BYTES = STAGE_OUT ? 4 * 32 * RK * 2 : 0;
  static constexpr int SMEM = kStages * kStageBytes + B_BYTES + 1024 + 256 + OUT_BYTES;
};

__device__ __forceinline__ uint16_t bf16_bits_rn(float x) {
  __nv_bfloat16 b = __float2bfloat16_rn(x);
  return *reinterpret_cast<uint16_t*>(&b);
}

template <int RK>
__global__ void __launch_bounds__(kThreads, 2) compress_tc_kernel(const __grid_constant__ CUtensorMap tmap, int N,
                                                                  int parts, const float* __restrict__ R,
                                                                  __nv_bfloat16* __restrict__ Kc, int nR,
                                                                  TokSrc tsrc, const __nv_bfloat16* __restrict__ Kg) {
  using C = CmpCfg<RK>;
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* Bsm = sm + kStages * kStageBytes;  // [split][half][RK rows][128 B], swizzled
  uint64_t* full = reinterpret_cast<uint64_t*>(Bsm + C::B_BYTES);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint4* outsm = reinterpret_cast<uint4*>(Bsm + C::B_BYTES + 256);  // [4 warps][32 rows][CPR]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.y, p = blockIdx.x;
  const int ntiles_all = (N + kTM - 1) / kTM;
  const int t_lo = (int)((long long)ntiles_all * p / parts);
  const int t_hi = (int)((long long)ntiles_all * (p + 1) / parts);
  const int nt = t_hi - t_lo;

  // ---- B = R^T split into hi/mid/lo bf16, K-major with the 128-byte swizzle
  const float* Ru = R + (size_t)(u % nR) * kDc * RK;  // nR < U: a shared (offline) rotation
  for (int e = threadIdx.x; e < kDc * RK; e += blockDim.x) {
    const int ch = e / RK, n = e % RK;   // coalesced read of R[ch][n]
    const float x = Ru[e];
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(h);
    const __nv_bfloat16 m = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(m);
    const __nv_bfloat16 l = __float2bfloat16_rn(r2);
    const int half = ch >> 6, c64 = ch & 63, chunk = c64 >> 3, within = (c64 & 7) * 2;
    const int off = half * C::B_HALF + n * 128 + ((chunk ^ (n & 7)) << 4) + within;
    *reinterpret_cast<__nv_bfloat16*>(Bsm + 0 * C::B_SPLIT + off) = h;
    *reinterpret_cast<__nv_bfloat16*>(Bsm + 1 * C::B_SPLIT + off) = m;
    *reinterpret_cast<__nv_bfloat16*>(Bsm + 2 * C::B_SPLIT + off) = l;
  }
  const bool gathered = tsrc.active();  // token list / per-unit lengths: cp.async producer
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], gathered ? 32 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
    if (!gathered) tc::prefetch_tmap(&tmap);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  fence_proxy_async();  // generic-proxy writes of B must be visible to the tensor core (async proxy)
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && gathered) {
    // all 32 lanes gather the tile's rows (tok_gather.cuh); rows past the unit's count are
    // zero-filled, so their K~ rows come out exactly 0
    const int nv = tsrc.valid(u, N);
    for (int i = 0; i < nt; ++i) {
      const int s = i % kStages;
      mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
      gather_tile_128x128(tsrc, Kg, u, N, nv, (t_lo + i) * kTM, sm + s * kStageBytes, kHalf, lane);
      cp_async_arrive_noinc(&full[s]);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < nt; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        unsigned char* dst = sm + s * kStageBytes;
        mbar_arrive_expect_tx(&full[s], kStageBytes);
        const int tok = (t_lo + i) * kTM;
        tc::tma_load_3d(dst, &tmap, 0, tok, u, &full[s], pol);
        tc::tma_load_3d(dst + kHalf, &tmap, 64, tok, u, &full[s], pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, RK, false, false);
      const uint32_t bbase = smem_u32(Bsm);
      for (int i = 0; i < nt; ++i) {
        const int s = i % kStages, a = i & 1;
        mbar_wait(&full[s], (i / kStages) & 1);
        if (gathered) fence_proxy_async();  // cp.async (generic proxy) writes -> tensor core
        mbar_wait(&tempty[a], ((i >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t abase = smem_u32(sm + s * kStageBytes);
        int first = 1;
#pragma unroll
        for (int kk = 0; kk < kDc / 16; ++kk) {
          const int half = kk >> 2, koff = (kk & 3) * 32;
          const uint64_t ad = tc::smem_desc(abase + half * kHalf + koff, 16, 1024, tc::SWZ_128B);
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            const uint64_t bd = tc::smem_desc(bbase + x * C::B_SPLIT + half * C::B_HALF + koff, 16, 1024,
                                              tc::SWZ_128B);
            tc::mma_bf16(tmem + a * RK, ad, bd, idesc, first ? 0u : 1u);
            first = 0;
          }
        }
        tc::commit(&empty[s]);
        tc::commit(&tfull[a]);
      }
    }
  } else {
    // ---- epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 = tokens of the tile
    const int q = warp & 3;
    const int m = 32 * q + lane;
    for (int i = 0; i < nt; ++i) {
      const int a = i & 1;
      mbar_wait(&tfull[a], (i >> 1) & 1);
      tc::fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + a * RK;
      const int tok = (t_lo + i) * kTM + m;
      __nv_bfloat16* dst = Kc + ((size_t)u * N + tok) * RK;
      // chunk swizzle of a staged row: the 8 rows one 128-byte shared-memory phase touches
      // land in 8 distinct 16-byte bank groups for the row-wise writes and the block reads
      auto swz = [](int row) { return (row / (8 / C::CPR)) & (C::CPR - 1); };
      uint4* stg = outsm + (warp - 2) * 32 * C::CPR;
#pragma unroll
      for (int b = 0; b < RK / 16; ++b) {
        uint32_t r[16];
        tc::ld_32x32b_x16(taddr + b * 16, r);
        tc::ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          pk[j] = (uint32_t)bf16_bits_rn(__uint_as_float(r[2 * j])) |
                  ((uint32_t)bf16_bits_rn(__uint_as_float(r[2 * j + 1])) << 16);
        if constexpr (C::STAGE_OUT) {
          stg[lane * C::CPR + ((2 * b) ^ swz(lane))] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          stg[lane * C::CPR + ((2 * b + 1) ^ swz(lane))] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        } else if (tok < N) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + b * 16);
          d4[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          d4[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      if constexpr (C::STAGE_OUT) {
        // the warp's 32 tokens are 32 consecutive rows of K~: one contiguous block, written
        // with every lane on consecutive 16-byte chunks (rows written lane-per-row put the
        // lanes r x 2 bytes apart)
        __syncwarp();
        const int tok0 = tok - lane;
        uint4* g4 = reinterpret_cast<uint4*>(Kc + ((size_t)u * N + tok0) * RK);
#pragma unroll
        for (int c = lane; c < 32 * C::CPR; c += 32) {
          const int row = c / C::CPR, ch = c % C::CPR;
          if (tok0 + row < N) g4[c] = stg[row * C::CPR + (ch ^ swz(row))];
        }
        __syncwarp();  // reads done before the next tile's staging
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[a]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

bool compress_tc_supported(int d, int r, bool bf16) {
  return bf16 && d == kDc && (r == 16 || r == 32 || r == 64 || r == 128);
}

template <int RK>
static int launch_compress_tc_r(int U, int N, const void* K, const float* R, void* Kc, cudaStream_t st,
                                int nR, const TokSrc& tsrc) {
  using C = CmpCfg<RK>;
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  if (!tsrc.active() && !encode_tmap_3d_bf16(&map, K, kDc, (uint64_t)N, (uint64_t)U, 64, kTM, 128)) return -2;
  static int attr_slot[kMaxDevices];
  once_per_device(attr_slot, [] {
    cudaFuncSetAttribute(compress_tc_kernel<RK>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    return 1;
  });
  const int ntiles = (N + kTM - 1) / kTM;
  int parts = (2 * kNumSMs + U - 1) / U;
  if (parts > ntiles) parts = ntiles;
  if (parts < 1) parts = 1;
  dim3 grid(parts, U);
  compress_tc_kernel<RK><<<grid, kThreads, C::SMEM, st>>>(map, N, parts, R, static_cast<__nv_bfloat16*>(Kc),
                                                          nR > 0 ? nR : U, tsrc,
                                                          static_cast<const __nv_bfloat16*>(K));
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_compress_tc(int U, int N, int r, const void* K, const float* R, void* Kc, cudaStream_t st,
                       int nR, const TokSrc& tsrc) {
  switch (r) {
    case 16: return launch_compress_tc_r<16>(U, N, K, R, Kc, st, nR, tsrc);
    case 32: return launch_compress_tc_r<32>(U, N, K, R, Kc, st, nR, tsrc);
    case 64: return launch_compress_tc_r<64>(U, N, K, R, Kc, st, nR, tsrc);
    case 128: return launch_compress_tc_r<128>(U, N, K, R, Kc, st, nR, tsrc);
  }
  return -2;
}

}  // namespace rk
