// decode_ring.cu -- host launcher of the CTA-ring GQA decode kernel (decode_ring.cuh).
#include <cstdlib>

#include "decode_common.cuh"

namespace rk {

#include "decode_ring.cuh"

// the CTA-ring GQA kernel (decode_ring.cuh): one CTA per SM over an equal contiguous range of
// the batch's tiles
template <int RK, int G>
static int launch_ring_cfg(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  using C = RingCfg<RK, G>;
  static_assert(C::SMEM <= 227 * 1024, "shared memory");
  RingPlan pl;
  pl.nvt = (a.N + C::TT - 1) / C::TT;
  pl.tpu = pl.nvt + (a.M + C::TX - 1) / C::TX;
  pl.T = (long long)a.U * pl.tpu;
  if ((long long)a.N + a.M >= (1LL << 30) || pl.T >= (1LL << 40)) return -3;
  const int sms = decode_num_sms();
  // CTAs: one per SM, fewer when a unit would span more CTAs than the merge's shared
  // (m, l) table holds (tiny batches, e.g. 4 units on 148 SMs)
  // at least ceil(tpu / div) tiles per CTA (default div 6: a unit spans <= 7 CTAs, so its
  // merge stays a few slots; tiny batches then use fewer SMs, each with a deeper stream --
  // Qwen b1 (4 units) 31.4 -> 18.4 us, b8 20.6 us; b32 / long unchanged; tools/time_decode.py)
  static int div_env = [] {
    const char* e = getenv("ROTATEK_RING_DIV");
    return e ? atoi(e) : 6;
  }();
  const long long minr_req = (pl.tpu + div_env - 1) / (div_env > 0 ? div_env : 6);
  long long cmax_ctas = pl.T / (minr_req > 0 ? minr_req : 1);
  if (cmax_ctas < 1) cmax_ctas = 1;
  for (pl.C = (int)(cmax_ctas < sms ? cmax_ctas : sms);; --pl.C) {
    const long long minr = pl.T / pl.C;  // >= 1 tile per CTA
    pl.cmax = (int)((pl.tpu + minr - 1) / minr) + 1;
    if (pl.cmax > pl.C) pl.cmax = pl.C;
    if (pl.cmax * a.G <= C::MLCAP || pl.C == 1) break;
  }
  // every CTA range must touch at most CAP units (the query table; all rotations up front)
  for (int c = 0; c < pl.C; ++c) {
    const long long kA = pl.start(c), kB = pl.start(c + 1);
    if (kB > kA && (kB - 1) / pl.tpu - kA / pl.tpu + 1 > C::CAP) return -3;
  }
  if ((size_t)a.U * pl.cmax * a.G * (kD + 4) * 4 > ws.partial_bytes) return -3;
  RingMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (!encode_tmap_3d_bf16(&maps.kc, a.Kc, RK, a.N, a.U, RK, C::TT, RK * 2)) return -2;
  if (!encode_tmap_3d_bf16(&maps.v, a.V, kD, a.N, a.U, 64, C::TT, 128)) return -2;
  if (a.M > 0) {
    if (!encode_tmap_3d_bf16_strided(&maps.kt, a.Kt, kD, a.M, a.U, a.Ms, 64, C::TX, 128)) return -2;
    if (!encode_tmap_3d_bf16_strided(&maps.vt, a.Vt, kD, a.M, a.U, a.Ms, 64, C::TX, 128)) return -2;
  }
  auto kern = decode_ring_kernel<RK, G>;
  static int attr_slot[kMaxDevices];
  once_per_device(attr_slot, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    return 1;
  });
  DecodeParams p{a.U, a.G, a.d, a.r, a.N, a.M, a.q, a.Kc, a.V, a.R, a.dmu, a.Kt, a.Vt,
                 a.scale * kLog2e, a.out, ws.counters, ws.partials, decode_trace_buffer(), 0, a.pout,
                 a.nR > 0 ? a.nR : a.U, nullptr, nullptr, a.overlap, a.Ms, a.nvu, a.ntu};
  // cooperative: the merging CTAs wait for their units' other contributors, so every CTA
  // must be resident (one per SM); plus programmatic serialization with ROTATEK_DECODE_OVERLAP
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.C);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.overlap ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, kern, maps, p, pl) != cudaSuccess) return -1;
  return 1;
}

template <int RK>
static int launch_ring_rk(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  switch (a.G) {
    case 2: return launch_ring_cfg<RK, 2>(a, ws, st);
    case 4: return launch_ring_cfg<RK, 4>(a, ws, st);
    case 7: return launch_ring_cfg<RK, 7>(a, ws, st);
    case 8: return launch_ring_cfg<RK, 8>(a, ws, st);
  }
  return -2;
}

int launch_ring(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  if (a.r == 32) return launch_ring_rk<32>(a, ws, st);
  if (a.r == 64) return launch_ring_rk<64>(a, ws, st);
  return -2;
}

}  // namespace rk
