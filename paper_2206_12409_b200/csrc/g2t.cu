// W2 = G2^T W1 for the three chi in one launch (Eq. 19 step 2), single
// right-hand side, without a split-K reduce launch.
//
// Per chi the product is tiny (r2 x n3l outputs, K = r1 n2 ~ 1200: 75 MFLOP) but its K is
// long, so the generic ZGEMM needs a 25-way split-K and a second launch to sum the partials
// (~20 us per chi, latency-bound).  Here a CTA owns an 8 x 8 output tile (beta, i3) and its
// 8 warps split K in eight contiguous ranges; each warp runs the 3M DMMA m8n8k4 over its
// range with its A (G2 columns, contiguous in K) and B (W1 columns, contiguous in K)
// fragments loaded straight from global memory, UNR k-steps in flight; the eight warp
// partials are summed by a fixed-order shared-memory tree and the tile is written once.
#include "common.cuh"
#include "kernels.cuh"

#include <cstdlib>

namespace vsie {
namespace {

constexpr int kG2Warps = 8;   // 16 measured no faster at cfg 2 and slower at cfg 4
constexpr int kG2Threads = 32 * kG2Warps;

__device__ __forceinline__ void dmma_g2(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// S > 1: split-K over the S CTAs of a thread-block cluster (grid z = chi * S + cluster rank):
// rank r takes K chunks [ksn r / S, ksn (r + 1) / S), its 8 warps split that range, and rank 0
// adds the S CTA partial tiles from the peers' shared memory (DSMEM, rank order: deterministic).
// Larger output tiles then keep the CTA count: 16 x 16 tiles with S = 4 read each operand from
// L2 half as often as 8 x 8 tiles with the same number of CTAs (the 8 x 8 kernel moves ~450 MB
// of L2 operand traffic per cfg 4 step, ~10 TB/s: its limiter)
template <int TM, int TN, int NW, int S>
__global__ void __launch_bounds__(32 * NW) k_g2t(const __grid_constant__ G2tArgs a) {
  __shared__ cplx red[NW / 2][64 * TM * TN];
  pdl_wait();
  const int b = blockIdx.z / S, kr = blockIdx.z % S;
  const int M = a.M[b], N = a.N, K = a.K[b];
  const int m0 = blockIdx.x * 8 * TM, n0 = blockIdx.y * 8 * TN;
  if (m0 >= M || n0 >= N) return;   // uniform per CTA (and per cluster)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ksn_all = (K + 3) / 4;
  const int kc0 = ksn_all * kr / S, ksn = ksn_all * (kr + 1) / S - kc0;
  const int ks0 = kc0 + ksn * warp / NW, ks1 = kc0 + ksn * (warp + 1) / NW;
  // A[m][k] = G2[k + K m] (op T of the column-major (r1 n2) x r2 core), B[k][n] = W1[k + K n]
  const cplx* Ar[TM];
  const cplx* Bc[TN];
#pragma unroll
  for (int i = 0; i < TM; ++i) Ar[i] = a.G2[b] + (int64_t)K * min(m0 + 8 * i + g, M - 1);   // clamped: discarded
#pragma unroll
  for (int j = 0; j < TN; ++j) Bc[j] = a.W1[b] + (int64_t)K * min(n0 + 8 * j + g, N - 1);
  double p1[TM][TN][2], p2[TM][TN][2], p3[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) p1[i][j][0] = p1[i][j][1] = p2[i][j][0] = p2[i][j][1] = p3[i][j][0] = p3[i][j][1] = 0;
  constexpr int UNR = TM * TN > 1 ? 5 : 10;
  for (int ks = ks0; ks < ks1; ks += UNR) {
    cplx av[UNR][TM], bv[UNR][TN];
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int k = 4 * (ks + q) + t;
      const bool ok = ks + q < ks1 && k < K;
#pragma unroll
      for (int i = 0; i < TM; ++i) av[q][i] = ok ? __ldg(Ar[i] + k) : cmk(0, 0);
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[q][j] = ok ? __ldcg(Bc[j] + k) : cmk(0, 0);
    }
#pragma unroll
    for (int q = 0; q < UNR; ++q)
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          dmma_g2(p1[i][j][0], p1[i][j][1], av[q][i].x, bv[q][j].x);
          dmma_g2(p2[i][j][0], p2[i][j][1], av[q][i].y, bv[q][j].y);
          dmma_g2(p3[i][j][0], p3[i][j][1], av[q][i].x + av[q][i].y, bv[q][j].x + bv[q][j].y);
        }
  }
  // lane holds C[8 i + g][8 j + 2 t + jj]; fixed-order tree over the warps
  cplx c[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
        c[i][j][jj] = cmk(p1[i][j][jj] - p2[i][j][jj], p3[i][j][jj] - p1[i][j][jj] - p2[i][j][jj]);
#pragma unroll
  for (int half = NW / 2; half >= 1; half >>= 1) {
    if (warp >= half && warp < 2 * half) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) red[warp - half][((i * TN + j) * 8 + g) * 8 + 2 * t + jj] = c[i][j][jj];
    }
    __syncthreads();
    if (warp < half) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
            c[i][j][jj] = cadd(c[i][j][jj], red[warp][((i * TN + j) * 8 + g) * 8 + 2 * t + jj]);
    }
    __syncthreads();
  }
  if (S > 1) {
    // the CTA partial (warp 0) into red[0] (free after the tree), then rank 0 sums the peers'
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) red[0][((i * TN + j) * 8 + g) * 8 + 2 * t + jj] = c[i][j][jj];
    }
    cluster_sync_all();
    if (kr == 0 && warp == 0) {
      for (int r = 1; r < S; ++r) {
        uint32_t base;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(base) : "r"((uint32_t)__cvta_generic_to_shared(&red[0][0])), "r"(r));
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              cplx v;
              const uint32_t addr = base + (uint32_t)((((i * TN + j) * 8 + g) * 8 + 2 * t + jj) * sizeof(cplx));
              asm volatile("ld.shared::cluster.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
              c[i][j][jj] = cadd(c[i][j][jj], v);
            }
      }
    }
    cluster_sync_all();   // the peers' shared memory stays alive until rank 0 has read it
  }
  if (warp == 0 && kr == 0) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int m = m0 + 8 * i + g, n = n0 + 8 * j + 2 * t + jj;
          if (m < M && n < N) a.W2[b][m + (int64_t)a.ldw[b] * n] = c[i][j][jj];
        }
  }
  pdl_trigger();
}

template <int TM, int TN, int S>
void launch_g2t_t(const G2tArgs& a, int mmax, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ceil_div(mmax, 8 * TM), (unsigned)ceil_div(a.N, 8 * TN), (unsigned)(a.nbatch * S));
  cfg.blockDim = dim3(32 * 8);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (S > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = S;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  VSIE_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_g2t<TM, TN, 8, S>, a));
  VSIE_CHECK_LAUNCH();
}

}  // namespace

// one CTA per 8 x 8 output tile, K split over its 8 warps; per 16 x 16 tile for large r2 n3;
// split-K over a 2-CTA cluster when the 8 x 8 tiles of the launch give < 512 CTAs.  Measured
// (profiles/r02c/ab_g2t_cluster.json, same box): cfg 2 (378 tiles) G2^T 22.9 -> 18.9 us, pair
// 0.1536 -> 0.1475-0.149 ms; cfg 4 (756 tiles) S = 2 45.8 vs 43.7 us, 16 x 16 tiles with S = 2
// / 4 (half the L2 operand traffic at >= as many CTAs) 54 / 48 us -- so the kernel is not bound
// by its L2 operand traffic; cfg 3 per-chi launches 16 x 16 S = 1 44.5 us vs 50-52 for S = 2 / 4;
// cfg 4 8 x 16 and 16 x 8 tiles without split-K (378 / 420 CTAs, 3/4 of the operand traffic)
// 46.1-46.4 / 45.8-46.1 vs 44.8 us (profiles/r02f/ab_g2t_tiles.json)
void launch_g2t(const G2tArgs& a, cudaStream_t st) {
  int mmax = 0;
  for (int b = 0; b < a.nbatch; ++b) mmax = std::max(mmax, a.M[b]);
  if (mmax == 0 || a.N == 0) return;
  const int64_t tiles8 = ceil_div(mmax, 8) * ceil_div(a.N, 8);
  // 16 x 16 tiles (a quarter of the L2 operand traffic) when a chi has many 8 x 8 tiles: cfg 3
  // (r2 = 137, n3 = 400: 900 tiles) pair 1.895 -> 1.831 ms; at cfg 4 (252 tiles) the 8 x 8
  // grid's parallelism wins (0.423 vs 0.432 ms)
  if (tiles8 >= 512) return launch_g2t_t<2, 2, 1>(a, mmax, st);
  if (tiles8 * a.nbatch < 512) return launch_g2t_t<1, 1, 2>(a, mmax, st);
  launch_g2t_t<1, 1, 1>(a, mmax, st);
}

}  // namespace vsie
