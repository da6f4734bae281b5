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

namespace vsie {
namespace {

constexpr int kG2Warps = 8;   // 16 measured no faster at cfg 2 and slower at cfg 4
constexpr int kG2Threads = 32 * kG2Warps;

__device__ __forceinline__ void dmma_g2(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kG2Threads) k_g2t(const __grid_constant__ G2tArgs a) {
  __shared__ cplx red[kG2Warps / 2][64];
  pdl_wait();
  const int b = blockIdx.z;
  const int M = a.M[b], N = a.N, K = a.K[b];
  const int m0 = blockIdx.x * 8, n0 = blockIdx.y * 8;
  if (m0 >= M || n0 >= N) return;   // uniform per CTA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ksn = (K + 3) / 4;
  const int ks0 = ksn * warp / kG2Warps, ks1 = ksn * (warp + 1) / kG2Warps;
  // A[m][k] = G2[k + K m] (op T of the column-major (r1 n2) x r2 core), B[k][n] = W1[k + K n]
  const int mrow = min(m0 + g, M - 1), ncol = min(n0 + g, N - 1);   // clamped rows / cols: discarded
  const cplx* __restrict__ Ar = a.G2[b] + (int64_t)K * mrow;
  const cplx* __restrict__ Bc = a.W1[b] + (int64_t)K * ncol;
  double p1[2] = {0, 0}, p2[2] = {0, 0}, p3[2] = {0, 0};
  constexpr int UNR = 10;
  for (int ks = ks0; ks < ks1; ks += UNR) {
    cplx av[UNR], bv[UNR];
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int k = 4 * (ks + q) + t;
      const bool ok = ks + q < ks1 && k < K;
      av[q] = ok ? __ldg(Ar + k) : cmk(0, 0);
      bv[q] = ok ? __ldcg(Bc + k) : cmk(0, 0);
    }
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      dmma_g2(p1[0], p1[1], av[q].x, bv[q].x);
      dmma_g2(p2[0], p2[1], av[q].y, bv[q].y);
      dmma_g2(p3[0], p3[1], av[q].x + av[q].y, bv[q].x + bv[q].y);
    }
  }
  // lane holds C[g][2 t + j]; fixed-order tree over the 8 warps
  cplx c[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) c[j] = cmk(p1[j] - p2[j], p3[j] - p1[j] - p2[j]);
#pragma unroll
  for (int half = kG2Warps / 2; half >= 1; half >>= 1) {
    if (warp >= half && warp < 2 * half) {
#pragma unroll
      for (int j = 0; j < 2; ++j) red[warp - half][g * 8 + 2 * t + j] = c[j];
    }
    __syncthreads();
    if (warp < half) {
#pragma unroll
      for (int j = 0; j < 2; ++j) c[j] = cadd(c[j], red[warp][g * 8 + 2 * t + j]);
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + g, n = n0 + 2 * t + j;
      if (m < M && n < N) a.W2[b][m + (int64_t)a.ldw[b] * n] = c[j];
    }
  }
  pdl_trigger();
}

// Forward G2 step Y2 = G2 Y3 (Eq. 17 step 3): M = r1 n2 rows, K = r2 (short), so
// no K split: warp w of a CTA owns the 8 x 8 tile (m-tile 8 blockIdx.x + w, n-tile
// blockIdx.y) over the whole K, 3M DMMA with fragments from L2 (A[m][k] = G2[m + M k],
// B[k][n] = Y3[k + K n]) and writes it once.
__global__ void __launch_bounds__(kG2Threads) k_g2n(const __grid_constant__ G2tArgs a) {
  pdl_wait();
  const int b = blockIdx.z;
  const int M = a.M[b], N = a.N, K = a.K[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = (blockIdx.x * kG2Warps + warp) * 8, n0 = blockIdx.y * 8;
  if (m0 < M && n0 < N) {
    const int g = lane >> 2, t = lane & 3;
    const int ksn = (K + 3) / 4;
    const int mrow = min(m0 + g, M - 1), ncol = min(n0 + g, N - 1);   // clamped: discarded
    const cplx* __restrict__ Am = a.G2[b] + mrow;                     // A[m][k] at Am[M k]
    const cplx* __restrict__ Bc = a.W1[b] + (int64_t)K * ncol;       // B[k][n] at Bc[k]
    double p1[2] = {0, 0}, p2[2] = {0, 0}, p3[2] = {0, 0};
    constexpr int UNR = 10;
    for (int ks = 0; ks < ksn; ks += UNR) {
      cplx av[UNR], bv[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int k = 4 * (ks + q) + t;
        const bool ok = k < K;
        av[q] = ok ? __ldg(Am + (int64_t)M * k) : cmk(0, 0);
        bv[q] = ok ? __ldcg(Bc + k) : cmk(0, 0);
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        dmma_g2(p1[0], p1[1], av[q].x, bv[q].x);
        dmma_g2(p2[0], p2[1], av[q].y, bv[q].y);
        dmma_g2(p3[0], p3[1], av[q].x + av[q].y, bv[q].x + bv[q].y);
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + g, n = n0 + 2 * t + j;
      if (m < M && n < N) a.W2[b][m + (int64_t)a.ldw[b] * n] = cmk(p1[j] - p2[j], p3[j] - p1[j] - p2[j]);
    }
  }
  pdl_trigger();
}

}  // namespace

void launch_g2n(const G2tArgs& a, cudaStream_t st) {
  int mmax = 0;
  for (int b = 0; b < a.nbatch; ++b) mmax = std::max(mmax, a.M[b]);
  if (mmax == 0 || a.N == 0) return;
  dim3 grid((unsigned)ceil_div(mmax, 8 * kG2Warps), (unsigned)ceil_div(a.N, 8), a.nbatch);
  launch_pdl(k_g2n, grid, dim3(kG2Threads), 0, st, a);
  VSIE_CHECK_LAUNCH();
}

void launch_g2t(const G2tArgs& a, cudaStream_t st) {
  int mmax = 0;
  for (int b = 0; b < a.nbatch; ++b) mmax = std::max(mmax, a.M[b]);
  if (mmax == 0 || a.N == 0) return;
  dim3 grid((unsigned)ceil_div(mmax, 8), (unsigned)ceil_div(a.N, 8), a.nbatch);
  launch_pdl(k_g2t, grid, dim3(kG2Threads), 0, st, a);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
