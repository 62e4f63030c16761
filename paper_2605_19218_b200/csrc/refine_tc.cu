// refine_tc.cu -- the fp64 refinement behind the fp32 Jacobi solvers (step 4), on the
// fp64 tensor cores and restricted to the columns select can keep.
//
// The fp32 solver returns V0 (columns in solver order) and lambda0.  Only the r largest
// eigenpairs leave calibrate (R_r, and delta_mu from it), so the refinement corrects the
// KC >= r + 8 candidate columns with the largest lambda0 (the margin keeps every column the
// refined ranking can select: lambda0 is accurate to ~1e-7 relative) and passes the others
// through:
//   order the columns by lambda0 (descending, ties -> lower index): candidates = first KC;
//   T = C_q V0[:, :KC];  B = V0^T T;  G = V0^T V0[:, :KC]            (fp64, DMMA m8n8k4)
//   lambda_j = B_jj / G_jj  (fp64 Rayleigh quotients, j < KC; lambda0 for the others)
//   W_ij = (B_ij - lambda_j G_ij) / (lambda_j - lambda_i)  (i != j, |W_ij| < kMaxW, else 0),
//   W_jj = (1 - G_jj) / 2                                   (first order of B x = lambda G x)
//   V[:, :KC] = V0[:, :KC] + V0 W.
// That is the same first-order step as refine_smem_kernel (calibrate.cu) on KC of the d columns:
// 4 GEMMs of d x d x KC instead of 4 of d^3.  One CTA (16 warps) per unit, V0 in shared memory
// as fp64 with a row stride = 4 (mod 16) doubles (conflict-free DMMA fragments); warp w owns
// output rows [8w, 8w + 8) of every GEMM.
#include "common.cuh"
#include "internal.h"

namespace rk {

namespace {
constexpr int kRtWarps = 16;
constexpr int kRtThreads = 32 * kRtWarps;
constexpr int kRtD = 128;
constexpr int kRtLdA = kRtD + 4;  // V0 row stride (doubles), = 4 (mod 16)
constexpr double kMaxW = 1e-3;    // as refine_smem_kernel: larger W = near-degenerate pair

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int KC>
struct RefTc {
  static constexpr int NT = KC / 8;
  static constexpr int LDT = KC + (20 - KC % 16) % 16;  // = 4 (mod 16)
  static constexpr size_t SMEM =
      ((size_t)kRtD * kRtLdA + (size_t)kRtD * LDT + 2 * kRtD) * sizeof(double) + 2 * kRtD * sizeof(int);
};
}  // namespace

template <int KC>
__global__ void __launch_bounds__(kRtThreads, 1) refine_tc_kernel(const double* __restrict__ cq,
                                                                 const float* __restrict__ v0g,
                                                                 float* __restrict__ lam,
                                                                 double* __restrict__ vout,
                                                                 const int32_t* __restrict__ jinfo) {
  using S = RefTc<KC>;
  constexpr int d = kRtD, LDA = kRtLdA, LDT = S::LDT, NT = S::NT;
  extern __shared__ __align__(16) double rts[];
  double* V0 = rts;                 // [d][LDA]  V0 with its columns in descending-lambda0 order
  double* T = V0 + d * LDA;         // [d][LDT]  C V0[:, :KC], then W, then the refined columns
  double* lp = T + d * LDT;         // [d]       lambda by position (refined for j < KC)
  double* l0 = lp + d;              // [d]       lambda0 in solver order
  int* perm = reinterpret_cast<int*>(l0 + d);  // [d] position -> solver column
  int* pos = perm + d;                         // [d] solver column -> position
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  if (jinfo[u] == -1) return;  // non-finite input: select zero-fills the unit
  const double* C = cq + (size_t)u * d * d;
  float* lu = lam + (size_t)u * d;
  // this lane's A fragments of step (1), C[8w + g][4i + c], requested before anything else so
  // their latency hides behind the ranking and the V0 staging (32 loads in flight per lane)
  double ca[d / 4];
  {
    const double* Crow = C + (size_t)(8 * w + g) * d + c;
#pragma unroll
    for (int i = 0; i < d / 4; ++i) ca[i] = __ldg(Crow + 4 * i);
  }

  // rank of every column by lambda0 (descending; ties -> lower index): sort-free and exact
  if (tid < d) l0[tid] = (double)lu[tid];
  __syncthreads();
  if (tid < d) {
    const double li = l0[tid];
    int rank = 0;
    for (int j = 0; j < d; ++j) {
      const double lj = l0[j];
      rank += (lj > li || (lj == li && j < tid)) ? 1 : 0;
    }
    perm[rank] = tid;
    pos[tid] = rank;
  }
  __syncthreads();
  // V0 (fp32, row-major, solver order) -> shared fp64, columns permuted
  const float* V0u = v0g + (size_t)u * d * d;
#pragma unroll
  for (int e = tid; e < d * d / 4; e += kRtThreads) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(V0u) + e);
    const int x = (4 * e) / d, o = (4 * e) % d;
    double* row = V0 + x * LDA;
    row[pos[o]] = v.x;
    row[pos[o + 1]] = v.y;
    row[pos[o + 2]] = v.z;
    row[pos[o + 3]] = v.w;
  }
  if (tid < d) lp[tid] = l0[perm[tid]];
  __syncthreads();

  // (1) T = C V0[:, :KC]: rows [8w, 8w + 8), C streamed from global (each element read once)
  {
    double acc[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < d; k0 += 4) {
      const double a = ca[k0 / 4];
      const double* Vk = V0 + (k0 + c) * LDA + g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt], a, Vk[8 * nt]);
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *reinterpret_cast<double2*>(T + (8 * w + g) * LDT + 8 * nt + 2 * c) = make_double2(acc[nt][0], acc[nt][1]);
  }
  __syncthreads();
  // (2) B = V0^T T and G = V0^T V0[:, :KC]: rows i in [8w, 8w + 8) (A[i][l] = V0[l][i])
  double bb[NT][2], gg[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) bb[nt][0] = bb[nt][1] = gg[nt][0] = gg[nt][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < d; k0 += 4) {
    const double a = V0[(k0 + c) * LDA + 8 * w + g];
    const double* Tk = T + (k0 + c) * LDT + g;
    const double* Vk = V0 + (k0 + c) * LDA + g;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      dmma884(bb[nt], a, Tk[8 * nt]);
      dmma884(gg[nt], a, Vk[8 * nt]);
    }
  }
  // Rayleigh quotients of the candidates: the diagonal entries (i == j)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (8 * w + g == 8 * nt + 2 * c + e) lp[8 * nt + 2 * c + e] = bb[nt][e] / gg[nt][e];
  __syncthreads();  // lp final; every warp is done reading T
  // (3) W in place of T (rows i = 8w + g)
  {
    const double bmax = fmax(fabs(lp[0]), fabs(lp[d - 1]));
    const int i = 8 * w + g;
    const double li = lp[i];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double wv[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * nt + 2 * c + e;
        const double lj = lp[j];
        const double num = bb[nt][e] - lj * gg[nt][e];
        const double gap = lj - li;
        if (i == j) wv[e] = 0.5 * (1.0 - gg[nt][e]);
        else if (fabs(gap) > 1e-12 * bmax && fabs(num) < kMaxW * fabs(gap)) wv[e] = num / gap;
        else wv[e] = 0.0;
      }
      *reinterpret_cast<double2*>(T + i * LDT + 8 * nt + 2 * c) = make_double2(wv[0], wv[1]);
    }
  }
  __syncthreads();
  // (4) V[:, :KC] = V0[:, :KC] + V0 W: rows x in [8w, 8w + 8)
  double acc[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const double2 v = *reinterpret_cast<const double2*>(V0 + (8 * w + g) * LDA + 8 * nt + 2 * c);
    acc[nt][0] = v.x;
    acc[nt][1] = v.y;
  }
#pragma unroll 4
  for (int k0 = 0; k0 < d; k0 += 4) {
    const double a = V0[(8 * w + g) * LDA + k0 + c];
    const double* Wk = T + (k0 + c) * LDT + g;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt], a, Wk[8 * nt]);
  }
  __syncthreads();  // every warp is done reading W
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
    *reinterpret_cast<double2*>(T + (8 * w + g) * LDT + 8 * nt + 2 * c) = make_double2(acc[nt][0], acc[nt][1]);
  __syncthreads();
  // outputs in solver order: refined candidates, V0 (exact fp32 values) for the rest
  double* Vo = vout + (size_t)u * d * d;
  for (int e = tid; e < d * d / 2; e += kRtThreads) {
    const int x = (2 * e) / d, o = (2 * e) % d;
    const int p0 = pos[o], p1 = pos[o + 1];
    const double v0 = p0 < KC ? T[x * LDT + p0] : V0[x * LDA + p0];
    const double v1 = p1 < KC ? T[x * LDT + p1] : V0[x * LDA + p1];
    reinterpret_cast<double2*>(Vo)[e] = make_double2(v0, v1);
  }
  if (tid < KC) lu[perm[tid]] = (float)lp[tid];
}

size_t refine_tc_smem_bytes(int kc) {
  return kc <= 40 ? RefTc<40>::SMEM : RefTc<72>::SMEM;
}

// candidates = r + 8 rounded to an instantiated size; 0 when r needs the full refinement
int refine_tc_candidates(int d, int r) {
  if (d != kRtD) return 0;
  if (r + 8 <= 40) return 40;
  if (r + 8 <= 72) return 72;
  return 0;
}

int launch_refine_tc(int U, int kc, const double* cq, const float* v32, float* lam, double* vecs,
                     const int32_t* jinfo, cudaStream_t st) {
  static int attr40[kMaxDevices], attr72[kMaxDevices];
  if (kc == 40) {
    once_per_device(attr40, [] {
      return cudaFuncSetAttribute(refine_tc_kernel<40>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)RefTc<40>::SMEM) == cudaSuccess ? 1 : 0;
    });
    refine_tc_kernel<40><<<U, kRtThreads, RefTc<40>::SMEM, st>>>(cq, v32, lam, vecs, jinfo);
  } else if (kc == 72) {
    once_per_device(attr72, [] {
      return cudaFuncSetAttribute(refine_tc_kernel<72>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)RefTc<72>::SMEM) == cudaSuccess ? 1 : 0;
    });
    refine_tc_kernel<72><<<U, kRtThreads, RefTc<72>::SMEM, st>>>(cq, v32, lam, vecs, jinfo);
  } else {
    return -1;
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rk
