// Fused transpose front of the TT apply, single right-hand side, batched over the three chi:
//   W1 = G1^T u      (Eq. 19 step 1)
//   W2 = G2^T W1     (Eq. 19 step 2)
// in ONE kernel, with W2 left as partial sums over blocks of 8 i2 values
// (W2p[blk][beta + r2 i3], summed in fixed block order by k_sum_w2p).
//
// Warp task = (chi, i2 block blk of 8, PG consecutive i3 planes).  For every plane the warp
// reduces the 8 voxel columns (i2 in blk, i3) of u over i1 on the FP64 tensor cores exactly
// as k_reduce_g1 (3M DMMA, G1 fragments in shared memory, the whole 8-column tile of u in
// flight), parks W1[a, i2] in warp-private shared memory, and then contracts the block's
// slice of G2 (r1 x 8 x r2, read through L1: the warps of a CTA share blk, so the slice is
// read from L2 about once per CTA) against the PG planes with DFMA, lanes over beta.
// Avoids W1's round trip, the G2^T split-K GEMM and its reduce launch; the FP64 pipe is
// shared by DMMA and DFMA, so the DFMA half costs what a DMMA would.
#include "common.cuh"
#include "kernels.cuh"

namespace vsie {
namespace {

constexpr int kAFWarps = 4;
constexpr int kAFThreads = 32 * kAFWarps;
constexpr int kPG = 4;          // i3 planes per warp task
constexpr int kBlk = 8;         // i2 values per block (one DMMA M tile of columns)

__device__ __forceinline__ void dmma_af(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(kAFThreads) k_adj12(const __grid_constant__ AdjFrontArgs a) {
  const int b = blockIdx.y;
  const int n1 = a.n1, n2 = a.n2, n3 = a.n3l, r1 = a.r1[b], r2 = a.r2[b];
  const int ks_n = (n1 + 3) / 4;
  extern __shared__ cplx af_smem[];
  cplx* Bf = af_smem;                                  // [ks_n][NT][32] fragments of G1
  cplx* W1s = af_smem + ks_n * NT * 32;                // [warp][8 NT][8][kPG] W1 tile per warp
  const cplx* __restrict__ G1 = a.G1[b];
  // G1 is a constant core: staged before waiting on the stream predecessor (PDL overlap)
  for (int e = threadIdx.x; e < ks_n * NT * 32; e += kAFThreads) {
    const int lane = e % 32, nt = (e / 32) % NT, ks = e / (32 * NT);
    const int k = 4 * ks + (lane & 3), n = 8 * nt + (lane >> 2);
    Bf[e] = (k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
  }
  __syncthreads();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  cplx* Ws = W1s + warp * (8 * NT) * kBlk * kPG;
  const double sgn = a.conj_u ? -1.0 : 1.0;
  const cplx* __restrict__ G2 = a.G2[b];
  const int nblk = (n2 + kBlk - 1) / kBlk;
  const int nq = (n3 + kPG - 1) / kPG;
  // CTA c of this chi: block blk = c % nblk and plane groups q = c / nblk + cpb j, taken by
  // its warps in turn (cpb = CTAs per block)
  const int cpb = max(1, (int)gridDim.x / nblk);
  const int blk = blockIdx.x % nblk;
  const int q0 = blockIdx.x / nblk;
  if (q0 >= cpb) return;
  const int i2 = blk * kBlk + g;
  const bool gok = i2 < n2;
  for (int q = q0 + cpb * warp; q < nq; q += cpb * kAFWarps) {
    // ---- W1 for the task's planes (G1^T on DMMA)
#pragma unroll 1
    for (int pp = 0; pp < kPG; ++pp) {
      const int i3 = q * kPG + pp;
      const bool cok = gok && i3 < n3;
      const cplx* __restrict__ U = a.u[b] + (cok ? (int64_t)n1 * (i2 + (int64_t)n2 * i3) : 0);
      double p1[NT][2], p2[NT][2], p3[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) p1[nt][0] = p1[nt][1] = p2[nt][0] = p2[nt][1] = p3[nt][0] = p3[nt][1] = 0;
      constexpr int UNR = 25;
      for (int ks = 0; ks < ks_n; ks += UNR) {
        cplx av[UNR];
#pragma unroll
        for (int qq = 0; qq < UNR; ++qq) {
          const int k = 4 * (ks + qq) + t;
          av[qq] = (cok && k < n1) ? __ldcs(U + k) : cmk(0, 0);
        }
#pragma unroll
        for (int qq = 0; qq < UNR; ++qq) {
          if (ks + qq < ks_n) {
            const double ar = av[qq].x, ai = sgn * av[qq].y, as = ar + ai;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const cplx bv = Bf[((ks + qq) * NT + nt) * 32 + lane];
              dmma_af(p1[nt][0], p1[nt][1], ar, bv.x);
              dmma_af(p2[nt][0], p2[nt][1], ai, bv.y);
              dmma_af(p3[nt][0], p3[nt][1], as, bv.x + bv.y);
            }
          }
        }
      }
      // lane holds W1[a = 8 nt + 2 t + j][column g]; park it as Ws[(a + r1 g) kPG + pp]
      // (rows a >= r1 and columns past n2 / planes past n3 are zero by construction)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int aa = 8 * nt + 2 * t + j;
          if (aa < r1)
            Ws[(aa + r1 * g) * kPG + pp] = cmk(p1[nt][j] - p2[nt][j], p3[nt][j] - p1[nt][j] - p2[nt][j]);
        }
    }
    __syncwarp();
    // ---- W2p[blk][beta + r2 i3] = sum_{a, g} G2[a, i2, beta] W1[a, i2, i3] (DFMA, lanes over beta)
    const int kmax = r1 * min(kBlk, n2 - blk * kBlk);
    for (int beta = lane; beta < r2; beta += 32) {
      const cplx* __restrict__ gcol = G2 + (int64_t)r1 * (blk * kBlk + (int64_t)n2 * beta);
      cplx acc[kPG];
#pragma unroll
      for (int pp = 0; pp < kPG; ++pp) acc[pp] = cmk(0, 0);
      // 8 G2 values (one 128-B line of this lane's column) in flight per step: the slice
      // is L1-resident after the first warp of the CTA, but the first touch goes to L2
      for (int k0 = 0; k0 < kmax; k0 += 8) {
        cplx gv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) gv[j] = k0 + j < kmax ? __ldg(gcol + k0 + j) : cmk(0, 0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (k0 + j < kmax) {
#pragma unroll
            for (int pp = 0; pp < kPG; ++pp) cfma(acc[pp], gv[j], Ws[(k0 + j) * kPG + pp]);
          }
        }
      }
      cplx* out = a.W2p[b] + (int64_t)blk * a.w2p_stride + beta;
#pragma unroll
      for (int pp = 0; pp < kPG; ++pp) {
        const int i3 = q * kPG + pp;
        if (i3 < n3) out[(int64_t)r2 * i3] = acc[pp];
      }
    }
    __syncwarp();   // Ws is rewritten by the next task
  }
  pdl_trigger();
}

// W2[chi][e] = sum_blk W2p[chi][blk][e], fixed block order
__global__ void __launch_bounds__(256) k_sum_w2p(const __grid_constant__ AdjFrontArgs a, int nblk) {
  pdl_wait();
  const int b = blockIdx.y;
  const int64_t n = (int64_t)a.r2[b] * a.n3l;
  for (int64_t e = blockIdx.x * 256LL + threadIdx.x; e < n; e += (int64_t)gridDim.x * 256) {
    const cplx* p = a.W2p[b] + e;
    cplx v[8];
    cplx s = cmk(0, 0);
    int k = 0;
    for (; k + 8 <= nblk; k += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + (int64_t)(k + j) * a.w2p_stride);
#pragma unroll
      for (int j = 0; j < 8; ++j) s = cadd(s, v[j]);
    }
    for (; k < nblk; ++k) s = cadd(s, __ldcg(p + (int64_t)k * a.w2p_stride));
    a.W2[b][e] = s;
  }
  pdl_trigger();
}

}  // namespace

bool adj_front_supported(int n1, int r1max) { return r1max >= 1 && r1max <= 16 && n1 >= 1 && n1 <= 256; }

void launch_adj_front(const AdjFrontArgs& a, cudaStream_t st) {
  int r1max = 0;
  for (int b = 0; b < a.nbatch; ++b) r1max = std::max(r1max, a.r1[b]);
  VSIE_REQUIRE(adj_front_supported(a.n1, r1max), VSIE_ERR_ARG, "adj_front: n1 > 256 or r1 > 16");
  const int NT = (r1max + 7) / 8;
  const int ks_n = (a.n1 + 3) / 4;
  const size_t smem = ((size_t)ks_n * NT * 32 + (size_t)kAFWarps * 8 * NT * kBlk * kPG) * sizeof(cplx);
  const int nblk = (a.n2 + kBlk - 1) / kBlk;
  const int nq = (a.n3l + kPG - 1) / kPG;
  const int cpb = std::max(1, (nq + kAFWarps - 1) / kAFWarps);   // one plane group per warp
  dim3 grid((unsigned)(nblk * cpb), a.nbatch);
  if (NT == 1) {
    static bool d = false;
    if (!d) {
      VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_adj12<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      d = true;
    }
    launch_pdl(k_adj12<1>, grid, dim3(kAFThreads), smem, st, a);
  } else {
    static bool d = false;
    if (!d) {
      VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_adj12<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      d = true;
    }
    launch_pdl(k_adj12<2>, grid, dim3(kAFThreads), smem, st, a);
  }
  VSIE_CHECK_LAUNCH();
  int64_t nmax = 0;
  for (int b = 0; b < a.nbatch; ++b) nmax = std::max<int64_t>(nmax, (int64_t)a.r2[b] * a.n3l);
  dim3 g2((unsigned)std::min<int64_t>(ceil_div(nmax, 256), 148 * 4), a.nbatch);
  launch_pdl(k_sum_w2p, g2, dim3(256), 0, st, a, nblk);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
