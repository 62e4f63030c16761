// decode_ring.cu -- host launcher of the CTA-ring GQA decode kernel (decode_ring.cuh).
#include <cstdlib>

#include "decode_common.cuh"

namespace rk {

#include "decode_ring.cuh"

static bool cluster_off() {  // experiments / A-B: ROTATEK_RING_NOCLUSTER=1 keeps the global merges
  static bool v = [] {
    const char* e = getenv("ROTATEK_RING_NOCLUSTER");
    return e && atoi(e) != 0;
  }();
  return v;
}

// CTA count of the ring kernel.  Ranges are equal contiguous tile ranges of the batch; the
// candidates are
//   * one per SM (at least ceil(tpu / div) tiles each: a unit then spans <= div + 1 CTAs, so
//     tiny batches use fewer SMs, each with a deeper stream -- Qwen b1 (4 units) 31.4 ->
//     18.4 us), whose range ends generally fall INSIDE units;
//   * U * k CTAs, k = min(sms / U, div): every unit cut into k equal pieces (range ends on unit
//     boundaries or equal fractions, all of a unit's contributors finish together);
//   * U / k CTAs (U > sms, k | U): k whole units per CTA, no cross-CTA merge at all.
// Estimate = max(largest range / per-SM stream rate, batch / HBM rate) + a merge penalty:
// a range end inside a unit leaves some unit with a contributor that reaches it only at the
// END of its range, so the unit's merge waits a GPU-scope publish (~4 us under the stream's
// load, traces); equal pieces (k <= 8) form one thread-block cluster per unit and merge
// through distributed shared memory (~0.5 us; ~2 us with a global last-arriver merge); whole
// units none.  Rates from tools/time_decode.py
// (qwen_b32_r32: 148 CTAs 36.9 us, 128 = one unit each 32.8 us, 64 = two units each 52.1 us ->
// ~57 GB/s per SM with the 8-stage ring; long_b16: 128 = halves 108.2 vs 148 111 us).
static int ring_ctas(int U, int tpu, int sms, int div, int stage_bytes, int cap) {
  const long long T = (long long)U * tpu;
  const double r_sm = 57e3, r_hbm = 6.9e6;  // bytes per us
  auto est = [&](long long Cc, double pen) {
    if (Cc < 1 || Cc > sms || Cc > T) return 1e30;  // every CTA holds >= 1 tile
    for (long long c = 0; c < Cc; ++c) {  // every range must touch at most `cap` units
      const long long kA = T * c / Cc, kB = T * (c + 1) / Cc;
      if (kB > kA && (kB - 1) / tpu - kA / tpu + 1 > cap) return 1e30;
    }
    const double t_sm = (double)((T + Cc - 1) / Cc) * stage_bytes / r_sm;
    const double t_hbm = (double)T * stage_bytes / r_hbm;
    return (t_sm > t_hbm ? t_sm : t_hbm) + pen;
  };
  const long long minr_req = (tpu + div - 1) / div;
  long long c0 = T / (minr_req > 0 ? minr_req : 1);
  if (c0 < 1) c0 = 1;
  if (c0 > sms) c0 = sms;
  const bool c0_clean = T % c0 == 0 && (c0 % U == 0 || U % c0 == 0);
  long long best = c0;
  double best_t = est(c0, c0_clean ? (c0 > U ? 2.0 : 0.0) : 4.0);
  auto consider = [&](long long Cc, double pen) {
    const double t = est(Cc, pen);
    if (t < best_t) { best_t = t; best = Cc; }
  };
  if (U <= sms) {
    // equal pieces: k <= 8 (one thread-block cluster per unit, DSMEM merge ~0.5 us)
    const int kmax = cluster_off() ? div : 8;
    int k = sms / U < kmax ? sms / U : kmax;
    if (k > tpu) k = tpu;  // >= 1 tile per piece
    consider((long long)U * k, k > 1 ? (cluster_off() ? 2.0 : 0.5) : 0.0);
  } else {
    for (int k = (U + sms - 1) / sms; k <= cap; ++k)
      if (U % k == 0) { consider(U / k, 0.0); break; }
  }
  static int c_env = [] {
    const char* e = getenv("ROTATEK_RING_C");  // experiments: force the CTA count
    return e ? atoi(e) : 0;
  }();
  if (c_env > 0 && c_env <= sms) best = c_env;
  return (int)best;
}

// the CTA-ring GQA kernel (decode_ring.cuh): one CTA per SM (or per unit / unit piece, see
// ring_ctas) over an equal contiguous range of the batch's tiles
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
  static int div_env = [] {
    const char* e = getenv("ROTATEK_RING_DIV");
    return e ? atoi(e) : 6;
  }();
  const int div = div_env > 0 ? div_env : 6;
  pl.C = ring_ctas(a.U, pl.tpu, sms, div, C::STAGE, C::CAP);
  for (;; --pl.C) {
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
  // equal-piece plan (every unit = k consecutive CTAs): one thread-block cluster per unit, the
  // pieces merged through distributed shared memory instead of a GPU-scope publish
  pl.clus = 0;
  {
    const int k = pl.C / a.U;
    if (k >= 2 && k <= 8 && pl.C == a.U * k && pl.tpu >= k && !cluster_off()) pl.clus = k;
  }
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
  // a plain launch (no CTA ever waits for another: the last contributor of a shared unit
  // merges it), plus programmatic serialization with ROTATEK_DECODE_OVERLAP
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.C);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (a.overlap) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (pl.clus > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = pl.clus;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cudaLaunchKernelEx(&cfg, kern, maps, p, pl) != cudaSuccess) {
    if (pl.clus <= 1) return -1;
    cudaGetLastError();  // the cluster shape could not be scheduled: plain launch, global merges
    pl.clus = 0;
    cfg.numAttrs = a.overlap ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, kern, maps, p, pl) != cudaSuccess) return -1;
  }
  return 1;
}

template <int RK>
static int launch_ring_rk(const DecodeArgs& a, const DecodeWs& ws, cudaStream_t st) {
  switch (a.G) {
    case 1: return launch_ring_cfg<RK, 1>(a, ws, st);
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
