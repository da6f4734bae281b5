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

template <int TM, int TN, int NW>
__global__ void __launch_bounds__(32 * NW) k_g2t(const __grid_constant__ G2tArgs a) {
  __shared__ cplx red[NW / 2][64 * TM * TN];
  pdl_wait();
  const int b = blockIdx.z;
  const int M = a.M[b], N = a.N, K = a.K[b];
  const int m0 = blockIdx.x * 8 * TM, n0 = blockIdx.y * 8 * TN;
  if (m0 >= M || n0 >= N) return;   // uniform per CTA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ksn = (K + 3) / 4;
  const int ks0 = ksn * warp / NW, ks1 = ksn * (warp + 1) / NW;
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
  if (warp == 0) {
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

}  // namespace

// one CTA per 8 x 8 output tile, K split over its 8 warps (16 x 16 / 8 x 16 tiles measured slower at
// cfgs 2 / 4), or per 16 x 16 tile for large r2 n3
void launch_g2t(const G2tArgs& a, cudaStream_t st) {
  int mmax = 0;
  for (int b = 0; b < a.nbatch; ++b) mmax = std::max(mmax, a.M[b]);
  if (mmax == 0 || a.N == 0) return;
  // 16 x 16 tiles (a quarter of the L2 operand traffic) when a chi has many 8 x 8 tiles: cfg 3
  // (r2 = 137, n3 = 400: 900 tiles) pair 1.895 -> 1.831 ms; at cfg 4 (252 tiles) the 8 x 8
  // grid's parallelism wins (0.423 vs 0.432 ms)
  if (ceil_div(mmax, 8) * ceil_div(a.N, 8) >= 512) {
    dim3 grid((unsigned)ceil_div(mmax, 16), (unsigned)ceil_div(a.N, 16), a.nbatch);
    launch_pdl(k_g2t<2, 2, 8>, grid, dim3(32 * 8), 0, st, a);
    VSIE_CHECK_LAUNCH();
    return;
  }
  dim3 grid((unsigned)ceil_div(mmax, 8), (unsigned)ceil_div(a.N, 8), a.nbatch);
  launch_pdl(k_g2t<1, 1, 8>, grid, dim3(32 * 8), 0, st, a);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
