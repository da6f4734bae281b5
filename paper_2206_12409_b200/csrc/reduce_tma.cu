// W1 = G1^T u for the three chi in one launch (Eq. 19 step 1), single
// right-hand side, u streamed by TMA.
//
// u^chi is column-major n1 x (n2 n3l) (i1 fastest), so every CTA's share -- the same column
// fraction [ncol s / ns, ncol (s + 1) / ns) of every chi -- is one contiguous byte range.  A
// producer warp streams it, chi after chi, in stages of 8 columns (one DMMA M tile,
// 16 n1 x 8 bytes) with one cp.async.bulk each; stage i is consumed by warp i % CW alone
// (one or two slots per warp), so loads and the FP64 work of different warps overlap instead
// of every warp loading, then computing (the latency-bound shape of k_reduce_g1).
//
// Arithmetic: W1[c][a] = sum_i1 G1[i1, a] u[i1, c].  The first 8 NTD values of a run on the
// FP64 tensor cores (3M DMMA m8n8k4 as in k_reduce_g1: lane (g, t) holds u[col g][4 ks + t],
// G1 fragments in shared memory); the REM <= 2 remaining values of a (r1 = 9, 10 at the
// measured ranks) run as exact DFMA on the same u registers and are summed over the four
// t lanes at the end.  DMMA and DFMA share one FP64 pipe, so this removes the
// padding of r1 = 10 to 16 (6 -> 3 DMMAs + 8 DFMAs per k-step).
#include "common.cuh"
#include "kernels.cuh"
#include "tma_ring.cuh"

namespace vsie {
namespace {
using namespace tma;

constexpr int kRTRing = 160 * 1024;

__device__ __forceinline__ void dmma_tma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NTD, int REM, int CW, int SPW>
__global__ void __launch_bounds__(32 * (CW + 1), 1) k_reduce_tma(const __grid_constant__ ReduceArgs a) {
  constexpr int kSlots = CW * SPW;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n1 = a.n1;
  const int ks_n = (n1 + 3) / 4;
  const int stage_elems = 8 * n1;
  cplx* ring = reinterpret_cast<cplx*>(smem);
  cplx* Bf = ring + (size_t)kSlots * stage_elems;             // [3][ks_n][NTD][32] DMMA fragments
  cplx* Gr = Bf + (size_t)3 * ks_n * (NTD > 0 ? NTD : 1) * 32;  // [3][4 ks_n][REM] DFMA columns
  __shared__ uint64_t full[kSlots], empty[kSlots];
  const int ns = gridDim.x, s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA column ranges start on multiples of 8 columns: every stage is one whole M tile and
  // (for n1 = 4 mod 8) its bulk copy starts on a 128-B boundary
  const int64_t c0 = s == 0 ? 0 : a.ncol * s / ns / 8 * 8;
  const int64_t c1 = s == ns - 1 ? a.ncol : a.ncol * (s + 1) / ns / 8 * 8;
  const int nc = (int)(c1 - c0);
  const int nst = (nc + 7) / 8;   // stages per chi (same for every chi)
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {
    // producer: u is the caller's input -- read only after the PDL wait
    pdl_wait();
    if (lane == 0) {
      int i = 0;
      for (int b = 0; b < a.nbatch; ++b) {
        for (int t = 0; t < nst; ++t, ++i) {
          const int slot = i % kSlots;
          if (i >= kSlots) mbar_wait(&empty[slot], ((i / kSlots) - 1) & 1);
          const int ncol = min(8, nc - 8 * t);
          const uint32_t bytes = (uint32_t)(16 * n1 * ncol);
          mbar_expect_tx(&full[slot], bytes);
          bulk_g2s(ring + (size_t)slot * stage_elems, a.u[b] + (int64_t)n1 * (c0 + 8 * t), bytes, &full[slot]);
        }
      }
    }
    return;
  }
  // constant cores: G1 of every chi staged by the consumer warps while the producer already
  // streams u (the fragments are needed only once the first stage has landed)
  for (int b = 0; b < a.nbatch; ++b) {
    const cplx* __restrict__ G1 = a.G1[b];
    const int r1 = a.r1[b];
    if (NTD > 0)
      for (int e = threadIdx.x; e < ks_n * NTD * 32; e += 32 * CW) {
        const int ln = e % 32, nt = (e / 32) % NTD, ks = e / (32 * NTD);
        const int k = 4 * ks + (ln & 3), n = 8 * nt + (ln >> 2);
        Bf[(size_t)b * ks_n * NTD * 32 + e] = (k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
      }
    for (int e = threadIdx.x; e < 4 * ks_n * REM; e += 32 * CW) {
      const int j = e % REM, k = e / REM, n = 8 * NTD + j;
      Gr[(size_t)b * 4 * ks_n * REM + e] = (k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * CW) : "memory");   // consumers only
  pdl_wait();
  const int g = lane >> 2, t = lane & 3;
  const double sgn = a.conj_u ? -1.0 : 1.0;
  const int total = a.nbatch * nst;
  for (int i = warp; i < total; i += CW) {
    const int b = i / nst, tt = i - b * nst;
    const int slot = i % kSlots;
    const int ncol = min(8, nc - 8 * tt);
    mbar_wait(&full[slot], (i / kSlots) & 1);
    const cplx* st = ring + (size_t)slot * stage_elems + (size_t)n1 * g;   // this lane's column
    const cplx* bf = Bf + (size_t)b * ks_n * (NTD > 0 ? NTD : 1) * 32;
    const cplx* gr = Gr + (size_t)b * 4 * ks_n * REM;
    double p1[NTD > 0 ? NTD : 1][2], p2[NTD > 0 ? NTD : 1][2], p3[NTD > 0 ? NTD : 1][2];
#pragma unroll
    for (int nt = 0; nt < NTD; ++nt) p1[nt][0] = p1[nt][1] = p2[nt][0] = p2[nt][1] = p3[nt][0] = p3[nt][1] = 0;
    cplx rem[REM > 0 ? REM : 1];
#pragma unroll
    for (int j = 0; j < REM; ++j) rem[j] = cmk(0, 0);
    const bool gok = g < ncol;   // columns past the CTA's range hold stale data: rows g discarded
    const int ks_end = a.diag == 1 ? 0 : ks_n;
#pragma unroll 4
    for (int ks = 0; ks < ks_end; ++ks) {
      const int k = 4 * ks + t;
      cplx av = (k < n1) ? st[k] : cmk(0, 0);
      av.y *= sgn;
#pragma unroll
      for (int nt = 0; nt < NTD; ++nt) {
        const cplx bv = bf[(ks * NTD + nt) * 32 + lane];
        dmma_tma(p1[nt][0], p1[nt][1], av.x, bv.x);
        dmma_tma(p2[nt][0], p2[nt][1], av.y, bv.y);
        dmma_tma(p3[nt][0], p3[nt][1], av.x + av.y, bv.x + bv.y);
      }
#pragma unroll
      for (int j = 0; j < REM; ++j) cfma(rem[j], gr[k * REM + j], av);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);   // every smem read of the stage is done
    const int r1 = a.r1[b];
    cplx* __restrict__ W = a.W1[b] + (int64_t)r1 * (c0 + 8 * tt + g);
    if (gok) {
#pragma unroll
      for (int nt = 0; nt < NTD; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int aa = 8 * nt + 2 * t + j;
          if (aa < r1) W[aa] = cmk(p1[nt][j] - p2[nt][j], p3[nt][j] - p1[nt][j] - p2[nt][j]);
        }
    }
#pragma unroll
    for (int j = 0; j < REM; ++j) {
      cplx v = rem[j];
      v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
      v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
      const int aa = 8 * NTD + j;
      if (gok && t == 0 && aa < r1) W[aa] = v;
    }
  }
  pdl_trigger();
}

template <int NTD, int REM, int CW, int SPW>
void launch_rt(const ReduceArgs& a, int ns, size_t smem, cudaStream_t st) {
  static size_t attr = 0;
  if (smem > attr) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_reduce_tma<NTD, REM, CW, SPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    attr = smem;
  }
  launch_pdl(k_reduce_tma<NTD, REM, CW, SPW>, dim3(ns), dim3(32 * (CW + 1)), smem, st, a);  // a.diag set by the caller
}

}  // namespace

namespace {
// ring geometry: consumer warps x slots per warp within the ring budget, at least two slots
// per warp (a single-buffered warp waits a full refill latency after every stage);
// VSIE_RT_CW overrides the number of consumer warps (2, 4 or 8).  false if it cannot fit.
bool rt_geometry(int n1, int r1max, int& ntd, int& rem, int& cw, int& spw, size_t& smem) {
  if (r1max > 18 || r1max < 1 || n1 < 1) return false;
  ntd = r1max / 8;
  rem = r1max % 8;
  if (rem > 2) {
    ntd += 1;
    rem = 0;
  }
  const int ks_n = (n1 + 3) / 4;
  const size_t stage = (size_t)16 * 8 * n1;
  const size_t fr = (size_t)3 * ks_n * std::max(ntd, 1) * 32 * 16 + (size_t)3 * 4 * ks_n * rem * 16;
  static const int cw_env = [] {
    const char* e = std::getenv("VSIE_RT_CW");
    return e ? std::atoi(e) : 0;
  }();
  cw = cw_env == 2 || cw_env == 4 || cw_env == 8 ? cw_env : 8;
  spw = 3;
  while (spw > 1 && cw * spw * stage > (size_t)kRTRing) --spw;
  while (cw > 2 && (cw * spw * stage > (size_t)kRTRing || (spw < 2 && cw_env == 0))) {
    cw /= 2;
    spw = 3;
    while (spw > 1 && cw * spw * stage > (size_t)kRTRing) --spw;
  }
  smem = cw * spw * stage + fr;
  return cw * spw * stage <= (size_t)kRTRing && smem <= 220 * 1024;
}
}  // namespace

bool reduce_tma_fits(int n1, int r1max) {
  int ntd, rem, cw, spw;
  size_t smem;
  return rt_geometry(n1, r1max, ntd, rem, cw, spw, smem);
}

// false when unsupported (the caller uses k_reduce_g1): single RHS only, r1 <= 18
bool launch_reduce_g1_tma(const ReduceArgs& a, cudaStream_t st) {
  int r1max = 0;
  for (int b = 0; b < a.nbatch; ++b) r1max = std::max(r1max, a.r1[b]);
  if (a.cols_per_rhs != a.ncol) return false;
  if (a.ncol == 0) return true;
  int ntd, rem, cw, spw;
  size_t smem;
  if (!rt_geometry(a.n1, r1max, ntd, rem, cw, spw, smem)) return false;
  const int ns = sm_count_dev();
  static const int diag = [] {
    const char* e = std::getenv("VSIE_RT_DIAG");
    return e ? std::atoi(e) : 0;
  }();
  ReduceArgs ad = a;
  ad.diag = diag;
#define VSIE_RT(NTD, REM)                                                                    \
  if (ntd == NTD && rem == REM) {                                                            \
    if (cw == 8 && spw == 3) launch_rt<NTD, REM, 8, 3>(ad, ns, smem, st);                     \
    else if (cw == 8 && spw == 2) launch_rt<NTD, REM, 8, 2>(ad, ns, smem, st);                \
    else if (cw == 8) launch_rt<NTD, REM, 8, 1>(ad, ns, smem, st);                            \
    else if (cw == 4 && spw == 3) launch_rt<NTD, REM, 4, 3>(ad, ns, smem, st);                \
    else if (cw == 4 && spw == 2) launch_rt<NTD, REM, 4, 2>(ad, ns, smem, st);                \
    else if (cw == 4) launch_rt<NTD, REM, 4, 1>(ad, ns, smem, st);                            \
    else if (spw == 3) launch_rt<NTD, REM, 2, 3>(ad, ns, smem, st);                           \
    else if (spw == 2) launch_rt<NTD, REM, 2, 2>(ad, ns, smem, st);                           \
    else launch_rt<NTD, REM, 2, 1>(ad, ns, smem, st);                                         \
    VSIE_CHECK_LAUNCH();                                                                     \
    return true;                                                                             \
  }
  VSIE_RT(0, 1) VSIE_RT(0, 2) VSIE_RT(1, 0) VSIE_RT(1, 1) VSIE_RT(1, 2) VSIE_RT(2, 0) VSIE_RT(2, 1) VSIE_RT(2, 2)
#undef VSIE_RT
  return false;
}

}  // namespace vsie
