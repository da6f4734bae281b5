// TT-core contraction kernels of the Z_bc apply: the per-chi chain
// kernels (the single-RHS streaming steps normally run as the batched TMA passes of
// pairg4.cu / segemv.cu, see apply.cu).
//
// Forward (Eq. 17), per chi:
//   y4 = G4 x            -> k_gemv_n_cp (r3 x m GEMV, HBM stream of G4)
//   Y3 = G3 y4           -> k_gemv_n_cp ((r2 n3) x r3 GEMV, HBM stream of G3)
//   Y2 = G2 Y3           -> zgemm      ((r1 n2) x r2 times r2 x n3)
//   y  = G1 Y2           -> k_expand_g1 (n1 x r1 times r1 x (n2 n3), coalesced voxel writes)
// Transpose (Eqs. 18-19), per chi, then summed over chi:
//   W1 = G1^T u          -> k_reduce_g1_tma (single RHS: TMA ring of whole column stages,
//                           warp pairs split k) / k_reduce_g1 (block RHS, small n1)
//   W2 = G2^T W1         -> zgemm (T)
//   z3 = G3^T W2         -> k_gemv_t   (column dot products, deterministic split over rows)
//   z  = sum_chi G4^T z3 -> k_gemv_t   (sum_batch)
// All split reductions are deterministic: partials are summed in a fixed order by a
// separate sum kernel, so results are bitwise reproducible run to run.
#include "kernels.cuh"
#include "dmma_tile.cuh"
#include "tma_ring.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>
#include <vector>

namespace vsie {

namespace {

constexpr int kThreads = 256;
constexpr int kXChunk = 512;

__device__ __forceinline__ cplx ldg_c(const cplx* p) { return __ldg(p); }

// Streaming 16-B load (evict-first).  asm volatile keeps a batch of these in program
// order ahead of the arithmetic that consumes them, so a thread really has U loads in
// flight (ptxas otherwise interleaves load/FMA pairs and keeps only two outstanding).
__device__ __forceinline__ cplx ld_stream(const cplx* p) {
  cplx v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// cp.async variant: thread t owns row t of its tile and keeps the next S - 1 columns of
// that row in flight as 16-B cp.async copies into its own smem slots (ring[slot][t]; no
// registers held, no barrier -- every slot is written and read by the same thread), so a
// CTA has S x blockDim x 16 B in flight: with 3 CTAs per SM ~190 KB per SM, the depth the
// loaded HBM latency (~5 us at 6 TB/s) needs.  x of the split staged in smem once.
template <int S>
__global__ void __launch_bounds__(320) k_gemv_n_cp(const __grid_constant__ GemvN a, cplx* __restrict__ partials,
                                                   int64_t rmax) {
  extern __shared__ __align__(16) cplx cp_smem[];
  pdl_wait();
  const int b = blockIdx.z;
  const int64_t R = a.R[b], C = a.C[b];
  const int T = blockDim.x, t = threadIdx.x;
  const int64_t row = (int64_t)blockIdx.y * T + t;
  const bool act = row < R;
  const int nsplit = gridDim.x, s = blockIdx.x;
  const int64_t c0 = C * s / nsplit, c1 = C * (s + 1) / nsplit;
  const int nc = (int)(c1 - c0);
  cplx* ring = cp_smem;                 // [S][T]
  cplx* xs = cp_smem + (size_t)S * T;   // [nc]
  const int64_t LD = a.lda[b] ? a.lda[b] : R;
  const cplx* __restrict__ p = a.A[b] + (act ? row : R - 1) + LD * c0;
  for (int j = t; j < nc; j += T) xs[j] = __ldcg(a.x[b] + c0 + j);
#pragma unroll
  for (int j = 0; j < S - 1; ++j) {
    if (j < nc) tc::cp_async16(ring + j * T + t, p + LD * j, 16);
    tc::cp_async_commit();
  }
  __syncthreads();   // xs visible
  cplx acc = cmk(0, 0), acc2 = cmk(0, 0);
  for (int j = 0; j < nc; ++j) {
    const int jn = j + S - 1;
    if (jn < nc) tc::cp_async16(ring + (jn % S) * T + t, p + LD * jn, 16);
    tc::cp_async_commit();
    tc::cp_async_wait<S - 1>();
    const cplx v = ring[(j % S) * T + t];
    if (j & 1) cfma(acc2, v, xs[j]); else cfma(acc, v, xs[j]);
  }
  pdl_trigger();
  acc = cadd(acc, acc2);
  if (!act) return;
  if (nsplit == 1)
    a.y[b][row] = acc;
  else
    partials[((int64_t)b * nsplit + s) * rmax + row] = acc;
}

struct SumArgs {
  cplx* y[3];
  int64_t n[3];
  int nbatch;
  bool conj_out;
};

// One warp per output: lanes stride over the splits, butterfly sum (fixed order).
__global__ void __launch_bounds__(kThreads) k_sum_partials_warp(const __grid_constant__ SumArgs a,
                                                                const cplx* __restrict__ partials, int nsplit,
                                                                int64_t stride) {
  pdl_wait();
  // tiny kernel: let the next (streaming) kernel launch now, so that it prefetches its
  // constant core while this one runs (it still waits for our completion to read us)
  pdl_trigger();
  const int b = blockIdx.y;
  const int64_t r = blockIdx.x * (int64_t)(kThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= a.n[b]) return;
  const cplx* p = partials + (int64_t)b * nsplit * stride + r;
  double sx = 0, sy = 0;
  for (int q = lane; q < nsplit; q += 32) {
    const cplx v = p[(int64_t)q * stride];
    sx += v.x;
    sy += v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
  }
  if (lane == 0) a.y[b][r] = cmk(sx, a.conj_out ? -sy : sy);
}

// y[b][r] = sum_q partials[(b * nsplit + q) * stride + r], fixed summation order
// (4 interleaved partial sums combined at the end): deterministic.

__global__ void __launch_bounds__(kThreads) k_sum_partials(const __grid_constant__ SumArgs a,
                                                           const cplx* __restrict__ partials, int nsplit,
                                                           int64_t stride) {
  pdl_wait();
  // tiny kernel: let the next (streaming) kernel launch now, so that it prefetches its
  // constant core while this one runs (it still waits for our completion to read us)
  pdl_trigger();
  const int b = blockIdx.y;
  const int64_t r = blockIdx.x * (int64_t)kThreads + threadIdx.x;
  if (r >= a.n[b]) return;
  const cplx* p = partials + (int64_t)b * nsplit * stride + r;
  cplx s0 = cmk(0, 0), s1 = s0, s2 = s0, s3 = s0;
  int q = 0;
  for (; q + 4 <= nsplit; q += 4) {
    s0 = cadd(s0, p[(int64_t)q * stride]);
    s1 = cadd(s1, p[(int64_t)(q + 1) * stride]);
    s2 = cadd(s2, p[(int64_t)(q + 2) * stride]);
    s3 = cadd(s3, p[(int64_t)(q + 3) * stride]);
  }
  for (; q < nsplit; ++q) s0 = cadd(s0, p[(int64_t)q * stride]);
  cplx v = cadd(cadd(s0, s1), cadd(s2, s3));
  if (a.conj_out) v.y = -v.y;
  a.y[b][r] = v;
}

constexpr int kWarps = kThreads / 32;
constexpr int kCPW = 2;                     // columns per warp
constexpr int kColsPerCta = kWarps * kCPW;  // 16
constexpr int kTU = 2;                      // row groups of 32 in flight per column

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y[c] = sum_r A[r + R c] x[r]  over rows [r0, r1) of this split: a warp owns kCPW
// columns, lanes stride the rows with kTU x kCPW independent 16-B streaming loads in
// flight; fixed-order lane sums (butterfly) -> deterministic.  In sum_batch mode the
// batches share the output columns (Eq. 18 sum over chi inside the kernel).
__global__ void __launch_bounds__(kThreads) k_gemv_t(const __grid_constant__ GemvT a, cplx* __restrict__ partials,
                                                     int64_t cmax) {
  pdl_wait();
  const bool conj_out = a.conj_out;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ct = blockIdx.x;
  const int nsplit = gridDim.y, s = blockIdx.y;
  const int bz = blockIdx.z;
  const int nb = a.sum_batch ? a.nbatch : 1;
  const int64_t Cout = a.C[a.sum_batch ? 0 : bz];
  if ((int64_t)ct * kColsPerCta >= Cout) return;
  const int64_t cbase = (int64_t)ct * kColsPerCta + warp * kCPW;
  cplx acc[kCPW];
#pragma unroll
  for (int j = 0; j < kCPW; ++j) acc[j] = cmk(0, 0);
  bool cok[kCPW];
#pragma unroll
  for (int j = 0; j < kCPW; ++j) cok[j] = cbase + j < Cout;
  for (int bb = 0; bb < nb; ++bb) {
    const int b = a.sum_batch ? bb : bz;
    const int64_t R = a.R[b];
    const int64_t r0 = R * s / nsplit, r1 = R * (s + 1) / nsplit;
    const cplx* __restrict__ A = a.A[b];
    const cplx* __restrict__ X = a.x[b];
    const cplx* __restrict__ col[kCPW];
#pragma unroll
    const int64_t LD = a.lda[b] ? a.lda[b] : R;
    for (int j = 0; j < kCPW; ++j) col[j] = A + LD * (cok[j] ? cbase + j : Cout - 1);
    int64_t r = r0 + lane;
    // software pipeline: the next kTU row groups are in flight while this batch is consumed
    if (r + 32 * (kTU - 1) < r1) {
      cplx v[kTU][kCPW], xv[kTU];
#pragma unroll
      for (int u = 0; u < kTU; ++u) {
        xv[u] = __ldg(X + r + 32 * u);
#pragma unroll
        for (int j = 0; j < kCPW; ++j) v[u][j] = ld_stream(col[j] + r + 32 * u);
      }
      r += 32 * kTU;
      for (; r + 32 * (kTU - 1) < r1; r += 32 * kTU) {
        cplx w[kTU][kCPW], xw[kTU];
#pragma unroll
        for (int u = 0; u < kTU; ++u) {
          xw[u] = __ldg(X + r + 32 * u);
#pragma unroll
          for (int j = 0; j < kCPW; ++j) w[u][j] = ld_stream(col[j] + r + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < kTU; ++u)
#pragma unroll
          for (int j = 0; j < kCPW; ++j) cfma(acc[j], v[u][j], xv[u]);
#pragma unroll
        for (int u = 0; u < kTU; ++u) {
          xv[u] = xw[u];
#pragma unroll
          for (int j = 0; j < kCPW; ++j) v[u][j] = w[u][j];
        }
      }
#pragma unroll
      for (int u = 0; u < kTU; ++u)
#pragma unroll
        for (int j = 0; j < kCPW; ++j) cfma(acc[j], v[u][j], xv[u]);
    }
    for (; r < r1; r += 32) {
      const cplx xv = __ldg(X + r);
#pragma unroll
      for (int j = 0; j < kCPW; ++j) cfma(acc[j], __ldcs(col[j] + r), xv);
    }
  }
  pdl_trigger();
#pragma unroll
  for (int j = 0; j < kCPW; ++j) {
    acc[j].x = warp_sum(acc[j].x);
    acc[j].y = warp_sum(acc[j].y);
  }
  if (lane < kCPW) {
    cplx v = acc[0];
#pragma unroll
    for (int j = 1; j < kCPW; ++j)
      if (lane == j) v = acc[j];
    const int64_t c = cbase + lane;
    if (c < Cout) {
      if (nsplit == 1)
        a.y[bz][c] = conj_out ? cconj(v) : v;
      else
        partials[((int64_t)bz * nsplit + s) * cmax + c] = v;
    }
  }
}

// ----------------------------------------------------------------------------- G1 steps on FP64 tensor cores
// Both G1 contractions are dense skinny GEMMs (K = r1 for the expansion, K = n1
// for the transpose reduction), so they run on the sm_100a FP64 tensor cores
// through mma.sync.m8n8k4.f64 (DMMA; tcgen05 has no f64 kind).  A complex
// product is 4 real DMMAs: C_re += A_re B_re - A_im B_im, C_im += A_re B_im + A_im B_re.
// Fragment layout of m8n8k4 (PTX ISA): lane = 4 g + t;  A[g][t], B[t][g],
// C[g][2 t + j] (j = 0, 1).
constexpr int kWarpsG1 = 8;
constexpr int kG1Threads = 32 * kWarpsG1;
constexpr int kColsPerWarp = 8;
constexpr int kColsPerCtaG1 = kColsPerWarp * kWarpsG1;   // 64 columns per CTA

__device__ __forceinline__ int64_t col_addr(int64_t c, int64_t cpr, int64_t ld, int n1) {
  if (c < cpr) return c * n1;  // single right-hand side: no division
  const int64_t rhs = c / cpr;
  return rhs * ld + (c - rhs * cpr) * n1;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// complex 8x8x4 block: (cr, ci) += A * B with A = (ar, ai), B = (br, bi) fragments
__device__ __forceinline__ void zmma(double (&cr)[2], double (&ci)[2], cplx a, cplx b) {
  dmma(cr[0], cr[1], a.x, b.x);
  dmma(cr[0], cr[1], -a.y, b.y);
  dmma(ci[0], ci[1], a.x, b.y);
  dmma(ci[0], ci[1], a.y, b.x);
}

// y[i1 + n1 c] = sum_a G1[i1 + n1 a] Y2[a + r1 c]: warp task = 8 columns x all i1;
// Y2 fragments in registers (KT k-steps), G1 fragments from shared memory; each
// 8 x 8 output tile is stored as 4 whole 128-B lines per warp instruction.
// KT DMMA k-steps cover k < 4 KT.  REMK = 1 (r1 = 9, 17): the remaining k = 4 KT runs as exact
// DFMA.  REMK = 2 (r1 = 10, 18): the two remaining k run as ONE extra k-step per output product
// pair with real and imaginary parts concatenated along k -- A = [Gr(k0) Gr(k1) Gi(k0) Gi(k1)],
// Re += A [Yr; Yr; -Yi; -Yi], Im += A [Yi; Yi; Yr; Yr] -- 2 DMMAs instead of the 3 of a padded
// 3M k-step (8 instead of 9 DMMAs per 8 x 8 tile at r1 = 10; the DMMA sub-pipe is this
// kernel's limiter, ncu 66% active with math-pipe throttle the top stall).  The ~12 FP64 adds
// per tile (operand sum, recombination) are NOT the limiter: a chained form with none --
// k1 = (Ar + Ai) Br, re = k1 - Ai (Br + Bi), im = k1 + Ar (Bi - Br) continuing the k1
// accumulator, operand sums staged in shared memory -- measured equal (39.3-39.6 us at cfg 4,
// four variants, profiles/r02d/ab_last_session.json), so the DMMA issue rate itself bounds it
template <int KT, int REMK>
__global__ void __launch_bounds__(kG1Threads) k_expand_g1(const __grid_constant__ ExpandArgs a) {
  const int b = blockIdx.y;
  const int n1 = a.n1, r1 = a.r1[b];
  const int mt = (n1 + 7) / 8;
  constexpr int KTA = KT > 0 ? KT : 1;
  // [mt][KT][32] fragments of G1, then (REMK 1) [8 mt] column 4 KT or (REMK 2) [mt][32] the
  // concatenated k-step's fragments
  extern __shared__ cplx Af[];
  cplx* Gk = Af + (size_t)mt * KTA * 32;
  const cplx* __restrict__ G1 = a.G1[b];
  // G1 is a constant core: staged before waiting on the producer of Y2 (PDL overlap), all
  // of a thread's loads in flight before its stores (a load -> store per element costs one
  // global latency per element, ~5 us of the kernel when nothing overlaps it)
  if (KT > 0) {
    const int tot = mt * KT * 32;
    for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * kG1Threads) {
      cplx v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = e0 + q * kG1Threads;
        const int lane = e % 32, ks = (e / 32) % KTA, m = e / (32 * KTA);
        const int i1 = 8 * m + (lane >> 2), k = 4 * ks + (lane & 3);
        v[q] = (e < tot && i1 < n1 && k < r1) ? __ldg(G1 + i1 + (int64_t)n1 * k) : cmk(0, 0);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (e0 + q * kG1Threads < tot) Af[e0 + q * kG1Threads] = v[q];
    }
  }
  if (REMK == 1)
    for (int e = threadIdx.x; e < 8 * mt; e += kG1Threads) {
      const int i1 = e, k = 4 * KT;
      Gk[e] = (i1 < n1 && k < r1) ? __ldg(G1 + i1 + (int64_t)n1 * k) : cmk(0, 0);
    }
  if (REMK == 2) {   // concatenated k-step fragments: Gc[m][lane] = (t < 2 ? Gr : Gi)[8 m + g][4 KT + (t & 1)]
    double* Gc = reinterpret_cast<double*>(Gk);
    for (int e = threadIdx.x; e < 32 * mt; e += kG1Threads) {
      const int ln = e % 32, i1 = 8 * (e / 32) + (ln >> 2), k = 4 * KT + (ln & 1);
      const cplx v = (i1 < n1 && k < r1) ? __ldg(G1 + i1 + (int64_t)n1 * k) : cmk(0, 0);
      Gc[e] = (ln & 2) ? v.y : v.x;
    }
  }
  __syncthreads();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  cplx* __restrict__ Y = a.y[b];
  // persistent: whole 8-column tasks strided over the warps (adjacent warps write adjacent
  // 25-KB blocks), or -- a.balanced, when the strided rounds would leave > 10% of the kernel
  // idle (cfg 3: 6000 tasks on 2368 warps = 2.53 rounds, expansion 61 -> 50 us) -- the (task, i1
  // tile) units split into one contiguous range per warp, equal to within one unit.  The next
  // task's Y2 values are loaded before the current task's DMMAs and stores
  const int64_t ntask = (a.ncol + kColsPerWarp - 1) / kColsPerWarp;
  const int64_t nwarp = (int64_t)gridDim.x * kWarpsG1, wi = (int64_t)blockIdx.x * kWarpsG1 + warp;
  const bool bal = a.balanced != 0;
  int64_t u0 = bal ? ntask * mt * wi / nwarp : 0;
  const int64_t u1 = bal ? ntask * mt * (wi + 1) / nwarp : 0;
  int64_t task = bal ? u0 / mt : wi;
  int m0 = bal ? (int)(u0 - task * mt) : 0;
  // DMMA fragments bf[ks] = Y2[4 ks + t][col g]; REMK 1: DFMA values yr[jj] = Y2[4 KT][col 2 t + jj];
  // REMK 2: yr[0] = Y2[4 KT + (t & 1)][col g] (the concatenated k-step's B values)
  auto load_bf = [&](int64_t tk, cplx (&bf)[KTA], cplx (&yr)[2]) {
    const int64_t c = tk * kColsPerWarp + g;
    const cplx* __restrict__ Y2 = a.Y2[b] + (int64_t)r1 * c;
#pragma unroll
    for (int ks = 0; ks < KT; ++ks) {
      const int k = 4 * ks + t;
      bf[ks] = (tk < ntask && c < a.ncol && k < r1) ? __ldg(Y2 + k) : cmk(0, 0);
    }
    if (REMK == 1) {
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int64_t cc = tk * kColsPerWarp + 2 * t + jj;
        const int k = 4 * KT;
        yr[jj] = (tk < ntask && cc < a.ncol && k < r1) ? __ldg(a.Y2[b] + (int64_t)r1 * cc + k) : cmk(0, 0);
      }
    }
    if (REMK == 2) {
      const int k = 4 * KT + (t & 1);
      yr[0] = (tk < ntask && c < a.ncol && k < r1) ? __ldg(Y2 + k) : cmk(0, 0);
    }
  };
  cplx bf[KTA], yr[2];
  if (bal && u0 >= u1) task = ntask;
  load_bf(task, bf, yr);
  while (task < ntask) {
    const int m1 = bal ? (int)min((int64_t)mt, m0 + (u1 - u0)) : mt;
    u0 += m1 - m0;
    const int64_t next = bal ? (u0 < u1 ? task + 1 : ntask) : task + nwarp;
    cplx bn[KTA], yn[2];
    load_bf(next, bn, yn);
    const int64_t c0 = task * kColsPerWarp;
    int64_t oaddr[2];
    bool ok[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t c = c0 + 2 * t + j;
      ok[j] = c < a.ncol;
      oaddr[j] = ok[j] ? col_addr(c, a.cols_per_rhs, a.ld_rhs, n1) : 0;
    }
    double bsum[KTA];
#pragma unroll
    for (int ks = 0; ks < KT; ++ks) bsum[ks] = bf[ks].x + bf[ks].y;
    // the concatenated k-step's B fragments (REMK 2)
    const double bre = (t & 2) ? -yr[0].y : yr[0].x, bim = (t & 2) ? yr[0].x : yr[0].y;
    for (int m = m0; m < m1; ++m) {
      // 3 real DMMAs per complex product: P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi)
      double p1[2] = {0, 0}, p2[2] = {0, 0}, p3[2] = {0, 0};
#pragma unroll
      for (int ks = 0; ks < KT; ++ks) {
        const cplx av = Af[(m * KTA + ks) * 32 + lane];
        dmma(p1[0], p1[1], av.x, bf[ks].x);
        dmma(p2[0], p2[1], av.y, bf[ks].y);
        dmma(p3[0], p3[1], av.x + av.y, bsum[ks]);
      }
      const int i1 = 8 * m + g;
      cplx o[2];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) o[jj] = cmk(p1[jj] - p2[jj], p3[jj] - p1[jj] - p2[jj]);
      if (REMK == 1) {
        const cplx gv = Gk[i1];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) cfma(o[jj], gv, yr[jj]);
      }
      if (REMK == 2) {
        const double ac = reinterpret_cast<const double*>(Gk)[m * 32 + lane];
        double er[2] = {0, 0}, ei[2] = {0, 0};
        dmma(er[0], er[1], ac, bre);
        dmma(ei[0], ei[1], ac, bim);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          o[jj].x += er[jj];
          o[jj].y += ei[jj];
        }
      }
      if (i1 < n1) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (ok[j]) __stcs(Y + oaddr[j] + i1, o[j]);
      }
    }
#pragma unroll
    for (int ks = 0; ks < KT; ++ks) bf[ks] = bn[ks];
    yr[0] = yn[0];
    yr[1] = yn[1];
    task = next;
    m0 = 0;
  }
  pdl_trigger();
}

// W1[a + r1 c] = sum_i1 G1[i1 + n1 a] u[i1 + n1 c] (conj(u) for op C): warp task =
// 8 columns x all a (NT n-tiles of 8); u fragments streamed from global (each
// lane 16 B, 64 contiguous bytes per column), G1 fragments from shared memory.
constexpr int kRedWarps = 4;                  // 128-thread CTAs: 3 resident per SM
constexpr int kRedThreads = 32 * kRedWarps;

// NT DMMA n-tiles cover a < 8 NT; the REM <= 2 values a = 8 NT .. 8 NT + REM - 1 (r1 = 9, 10,
// 17, 18) run as exact DFMA on the same u registers (DMMA and DFMA share the FP64 pipe, so
// padding r1 = 10 to 16 or 17 to 24 would cost 1.6x / 1.4x the FP64 cycles)
template <int NT, int REM>
__global__ void __launch_bounds__(kRedThreads) k_reduce_g1(const __grid_constant__ ReduceArgs a) {
  const int b = blockIdx.y;
  const int n1 = a.n1, r1 = a.r1[b];
  const int ks_n = (n1 + 3) / 4;
  constexpr int NTA = NT > 0 ? NT : 1;
  extern __shared__ cplx Bf[];   // [ks_n][NT][32] fragments of G1, then [4 ks_n][REM] columns
  cplx* Gr = Bf + (size_t)ks_n * NTA * 32;
  const cplx* __restrict__ G1 = a.G1[b];
  // G1 is a constant core: staged before waiting on the stream predecessor (PDL overlap),
  // all of a thread's loads in flight before its stores
  if (NT > 0) {
    const int tot = ks_n * NT * 32;
    for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * kRedThreads) {
      cplx v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = e0 + q * kRedThreads;
        const int lane = e % 32, nt = (e / 32) % NTA, ks = e / (32 * NTA);
        const int k = 4 * ks + (lane & 3), n = 8 * nt + (lane >> 2);
        v[q] = (e < tot && k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (e0 + q * kRedThreads < tot) Bf[e0 + q * kRedThreads] = v[q];
    }
  }
  for (int e = threadIdx.x; e < 4 * ks_n * REM; e += kRedThreads) {
    const int j = e % (REM > 0 ? REM : 1), k = e / (REM > 0 ? REM : 1), n = 8 * NT + j;
    Gr[e] = (k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
  }
  __syncthreads();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const double sgn = a.conj_u ? -1.0 : 1.0;
  // persistent: warp tasks of 8 columns x all i1, UNR k-steps (100 rows) of loads in flight
  const int64_t ntask = (a.ncol + kColsPerWarp - 1) / kColsPerWarp;
  for (int64_t task = (int64_t)blockIdx.x * kRedWarps + warp; task < ntask; task += (int64_t)gridDim.x * kRedWarps) {
    const int64_t cg = task * kColsPerWarp + g;
    const bool cok = cg < a.ncol;
    const cplx* __restrict__ U = a.u[b] + (cok ? col_addr(cg, a.cols_per_rhs, a.ld_rhs, n1) : 0);
    // 3 real DMMAs per complex product (P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi))
    double p1[NTA][2], p2[NTA][2], p3[NTA][2];
#pragma unroll
    for (int nt = 0; nt < NTA; ++nt) p1[nt][0] = p1[nt][1] = p2[nt][0] = p2[nt][1] = p3[nt][0] = p3[nt][1] = 0;
    cplx rem[REM > 0 ? REM : 1];
#pragma unroll
    for (int j = 0; j < REM; ++j) rem[j] = cmk(0, 0);
    constexpr int UNR = 25;   // n1 <= 100: the whole column tile in flight at once
    for (int ks = 0; ks < ks_n; ks += UNR) {
      cplx av[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int k = 4 * (ks + q) + t;
        av[q] = (cok && k < n1) ? __ldcs(U + k) : cmk(0, 0);
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        if (ks + q < ks_n) {
          const double ar = av[q].x, ai = sgn * av[q].y, as = ar + ai;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const cplx bv = Bf[((ks + q) * NTA + nt) * 32 + lane];
            dmma(p1[nt][0], p1[nt][1], ar, bv.x);
            dmma(p2[nt][0], p2[nt][1], ai, bv.y);
            dmma(p3[nt][0], p3[nt][1], as, bv.x + bv.y);
          }
#pragma unroll
          for (int j = 0; j < REM; ++j) cfma(rem[j], Gr[(4 * (ks + q) + t) * REM + j], cmk(ar, ai));
        }
      }
    }
    // lane holds rows c = c0 + g, columns a = 8 nt + 2 t + j
    cplx* __restrict__ W = a.W1[b] + (int64_t)r1 * cg;
    if (cok) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int aa = 8 * nt + 2 * t + j;
          if (aa < r1) W[aa] = cmk(p1[nt][j] - p2[nt][j], p3[nt][j] - p1[nt][j] - p2[nt][j]);
        }
    }
#pragma unroll
    for (int j = 0; j < REM; ++j) {
      cplx v = rem[j];   // sum over the four k lanes t of this column
      v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
      v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
      const int aa = 8 * NT + j;
      if (cok && t == 0 && aa < r1) W[aa] = v;
    }
  }
  pdl_trigger();
}

// G1^T reduction fed by a TMA ring (single RHS: the columns of one chi are contiguous in u,
// so a stage of 8 q consecutive columns is ONE bulk copy of 8 q n1 x 16 B).  One producer
// warp keeps every free stage in flight; each stage is consumed by a PAIR of warps that split
// its k range in halves (task j -> slot j % ns, pair j % npairs) and only compute: no register
// is held by a load, so the FP64 pipe (DMMA + the DFMA remainder share it, ~0.7 of it at the
// HBM rate for r1 = 10) runs under the stream instead of between load batches.  Once both
// halves are done with the stage's u data, the upper half's partial sums go through the
// stage buffer itself to the lower half, which adds them (fixed order: lower + upper) and
// stores W1, then frees the slot.
constexpr int kRtPairs = 8;
constexpr int kRtThreads = 32 * (2 * kRtPairs + 1);

// stages L2-prefetched beyond the ring (cfg 4 pair 0.438 -> 0.422 ms with 1-3, slower with 8)
constexpr int kG1tPrefetch = 2;

template <int NT, int REM, bool CJ>
__global__ void __launch_bounds__(kRtThreads, 1) k_reduce_g1_tma(const __grid_constant__ ReduceArgs a, int q, int ns,
                                                                  int64_t stage_off) {
  const int b = blockIdx.y;
  const int n1 = a.n1, r1 = a.r1[b];
  const int ks_n = (n1 + 3) / 4;
  constexpr int NTA = NT > 0 ? NT : 1, RA = REM > 0 ? REM : 1;
  extern __shared__ __align__(128) unsigned char sm_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm_raw);   // [ns]
  uint64_t* empty = full + 16;                            // [ns]
  cplx* Bf = reinterpret_cast<cplx*>(sm_raw + 256);       // [ks_n][NT][32] fragments of G1
  cplx* Gr = Bf + (size_t)ks_n * NTA * 32;                // [4 ks_n][REM] columns a >= 8 NT
  cplx* stg = reinterpret_cast<cplx*>(sm_raw + stage_off);
  const int64_t cps = 8LL * q;                            // columns per stage
  const int64_t stage_elems = cps * n1;
  const int64_t nst = (a.ncol + cps - 1) / cps;
  const cplx* __restrict__ G1 = a.G1[b];
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      tma::mbar_init(full + s, 1);
      tma::mbar_init(empty + s, q);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (NT > 0)
    for (int e = threadIdx.x; e < ks_n * NT * 32; e += blockDim.x) {
      const int lane = e % 32, nt = (e / 32) % NTA, ks = e / (32 * NTA);
      const int k = 4 * ks + (lane & 3), n = 8 * nt + (lane >> 2);
      Bf[e] = (k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
    }
  for (int e = threadIdx.x; e < 4 * ks_n * REM; e += blockDim.x) {
    const int j = e % RA, k = e / RA, n = 8 * NT + j;
    Gr[e] = (k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == (int)(blockDim.x / 32) - 1) {
    // producer: u is the caller's input -- read only after the PDL wait
    pdl_wait();
    if (lane == 0) {
      const cplx* __restrict__ U = a.u[b];
      int j = 0;
      // L2 prefetch pf stages beyond the ring: more bytes in flight than the shared memory
      // holds (the stage a slot is refilled with is then an L2 hit)
      constexpr int pf = kG1tPrefetch;
      for (int64_t tp = blockIdx.x; tp < nst && tp < blockIdx.x + (int64_t)pf * gridDim.x; tp += gridDim.x) {
        const int64_t c0 = tp * cps;
        tma::bulk_prefetch_l2(U + c0 * n1, (uint32_t)(min(cps, a.ncol - c0) * n1 * (int64_t)sizeof(cplx)));
      }
      for (int64_t t = blockIdx.x; t < nst; t += gridDim.x, ++j) {
        const int slot = j % ns;
        if (j >= ns) tma::mbar_wait(empty + slot, ((j / ns) - 1) & 1);
        const int64_t c0 = t * cps;
        const int64_t nc = min(cps, a.ncol - c0);
        const uint32_t bytes = (uint32_t)(nc * n1 * (int64_t)sizeof(cplx));
        tma::mbar_expect_tx(full + slot, bytes);
        tma::bulk_g2s(stg + slot * stage_elems, U + c0 * n1, bytes, full + slot);
        const int64_t tn = t + (int64_t)pf * gridDim.x;
        if (tn < nst) {
          const int64_t cn = tn * cps;
          tma::bulk_prefetch_l2(U + cn * n1, (uint32_t)(min(cps, a.ncol - cn) * n1 * (int64_t)sizeof(cplx)));
        }
      }
    }
    pdl_trigger();
    return;
  }
  // consumer groups of 2 q warps (warp pair (tile, half) per 8-column tile of a stage): at
  // most ns groups, so that the stage a group waits for is never two ring phases ahead of the
  // producer (the group's previous task was j - ngroups >= j - ns)
  const int gsz = 2 * q;
  const int ngroups = (int)(blockDim.x / 32 - 1) / gsz;   // launched with 2 q ngroups + 1 warps
  const int grp = warp / gsz, tile = (warp % gsz) >> 1, half = warp & 1;
  const int ksh = (ks_n + 1) / 2;
  const int ks0 = half ? ksh : 0, ks1 = half ? ks_n : ksh;
  const int g = lane >> 2, t4 = lane & 3;
  int j = grp;
  for (int64_t t = blockIdx.x + (int64_t)grp * gridDim.x; t < nst; t += (int64_t)ngroups * gridDim.x, j += ngroups) {
    const int slot = j % ns;
    tma::mbar_wait(full + slot, (j / ns) & 1);
    cplx* S = stg + slot * stage_elems;
    {
      const int64_t cg = t * cps + 8 * tile + g;
      const cplx* __restrict__ col = S + (int64_t)(8 * tile + g) * n1;
      double p1[NTA][2], p2[NTA][2], p3[NTA][2];
#pragma unroll
      for (int nt = 0; nt < NTA; ++nt) p1[nt][0] = p1[nt][1] = p2[nt][0] = p2[nt][1] = p3[nt][0] = p3[nt][1] = 0;
      cplx rem[RA];
#pragma unroll
      for (int jj = 0; jj < RA; ++jj) rem[jj] = cmk(0, 0);
#pragma unroll 5
      for (int ks = ks0; ks < ks1; ++ks) {
        const int k = 4 * ks + t4;
        const cplx av = k < n1 ? col[k] : cmk(0, 0);
        const double ar = av.x, ai = CJ ? -av.y : av.y, as = ar + ai;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const cplx bv = Bf[(ks * NTA + nt) * 32 + lane];
          dmma(p1[nt][0], p1[nt][1], ar, bv.x);
          dmma(p2[nt][0], p2[nt][1], ai, bv.y);
          dmma(p3[nt][0], p3[nt][1], as, bv.x + bv.y);
        }
#pragma unroll
        for (int jj = 0; jj < REM; ++jj) cfma(rem[jj], Gr[k * REM + jj], cmk(ar, ai));
      }
      // both halves are done with this tile's u: the upper half's partials go through the
      // stage buffer (tile 8 columns x n1 >= 32 lanes x 6 NT + 2 REM doubles, checked by the host) to the lower half
      double* xch = reinterpret_cast<double*>(S + (int64_t)8 * tile * n1);
      asm volatile("bar.sync %0, 64;" ::"r"(1 + grp * q + tile) : "memory");
      if (half) {
#pragma unroll
        for (int nt = 0; nt < NTA; ++nt)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            xch[(6 * nt + jj) * 32 + lane] = p1[nt][jj];
            xch[(6 * nt + 2 + jj) * 32 + lane] = p2[nt][jj];
            xch[(6 * nt + 4 + jj) * 32 + lane] = p3[nt][jj];
          }
#pragma unroll
        for (int jj = 0; jj < RA; ++jj) {
          xch[(6 * NTA + 2 * jj) * 32 + lane] = rem[jj].x;
          xch[(6 * NTA + 2 * jj + 1) * 32 + lane] = rem[jj].y;
        }
      }
      asm volatile("bar.sync %0, 64;" ::"r"(1 + grp * q + tile) : "memory");
      if (!half) {
#pragma unroll
      for (int nt = 0; nt < NTA; ++nt)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          p1[nt][jj] += xch[(6 * nt + jj) * 32 + lane];
          p2[nt][jj] += xch[(6 * nt + 2 + jj) * 32 + lane];
          p3[nt][jj] += xch[(6 * nt + 4 + jj) * 32 + lane];
        }
#pragma unroll
      for (int jj = 0; jj < RA; ++jj) {
        rem[jj].x += xch[(6 * NTA + 2 * jj) * 32 + lane];
        rem[jj].y += xch[(6 * NTA + 2 * jj + 1) * 32 + lane];
      }
      const bool cok = cg < a.ncol;
      cplx* __restrict__ W = a.W1[b] + (int64_t)r1 * cg;
      if (cok) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int aa = 8 * nt + 2 * t4 + jj;
            if (aa < r1) W[aa] = cmk(p1[nt][jj] - p2[nt][jj], p3[nt][jj] - p1[nt][jj] - p2[nt][jj]);
          }
      }
#pragma unroll
      for (int jj = 0; jj < REM; ++jj) {
        cplx v = rem[jj];
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
        const int aa = 8 * NT + jj;
        if (cok && t4 == 0 && aa < r1) W[aa] = v;
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(empty + slot);   // one arrival per tile (count q)
      }
    }
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(kThreads) k_sum3(const cplx* __restrict__ in, int64_t chi_stride, int64_t ld_in,
                                                   int64_t rows, int k, cplx* __restrict__ out, int64_t ld_out,
                                                   bool conj_out) {
  pdl_wait();
  // tiny kernel: let the next (streaming) kernel launch now, so that it prefetches its
  // constant core while this one runs (it still waits for our completion to read us)
  pdl_trigger();
  const int64_t n = rows * k;
  for (int64_t e = blockIdx.x * (int64_t)kThreads + threadIdx.x; e < n; e += (int64_t)gridDim.x * kThreads) {
    const int64_t j = e / rows, i = e - j * rows;
    const cplx* p = in + i + ld_in * j;
    cplx v = cadd(cadd(p[0], p[chi_stride]), p[2 * chi_stride]);
    if (conj_out) v.y = -v.y;
    out[i + ld_out * j] = v;
  }
}

int pick_splits(int64_t other_ctas, int64_t len, int min_len, int max_splits, int64_t target) {
  int64_t sp = target / std::max<int64_t>(1, other_ctas);
  sp = std::min<int64_t>(sp, len / std::max(1, min_len));
  sp = std::min<int64_t>(sp, max_splits);
  return (int)std::max<int64_t>(1, sp);
}

// resident blocks per SM of a kernel at a block size (cached)
int gemv_occupancy(const void* fn, int threads) {
  static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
  for (auto& e : cache)
    if (e.first.first == fn && e.first.second == threads) return e.second;
  int occ = 1;
  VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0));
  occ = std::max(1, occ);
  cache.push_back({{fn, threads}, occ});
  return occ;
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

int sm_count_dev() { return sm_count(); }

void launch_gemv_sum(const GemvN& a, cplx* partials, int ns, int64_t rmax, cudaStream_t st) {
  if (ns <= 1) return;
  SumArgs sa{};
  sa.nbatch = a.nbatch;
  for (int b = 0; b < a.nbatch; ++b) {
    sa.y[b] = a.y[b];
    sa.n[b] = a.R[b];
  }
  if (ns >= 16) {
    dim3 g2((unsigned)ceil_div(rmax, kThreads / 32), a.nbatch);
    launch_pdl(k_sum_partials_warp, g2, dim3(kThreads), 0, st, sa, (const cplx*)partials, ns, rmax);
  } else {
    dim3 g2((unsigned)ceil_div(rmax, kThreads), a.nbatch);
    launch_pdl(k_sum_partials, g2, dim3(kThreads), 0, st, sa, (const cplx*)partials, ns, rmax);
  }
  VSIE_CHECK_LAUNCH();
}

void launch_gemv_n(const GemvN& a, cplx* partials, int64_t partials_cap, int max_splits, cudaStream_t st) {
  int64_t rmax = 0, cmax = 0;
  for (int b = 0; b < a.nbatch; ++b) {
    rmax = std::max(rmax, a.R[b]);
    cmax = std::max(cmax, a.C[b]);
  }
  if (rmax == 0) return;
  {
    constexpr int S = 16;
    const int T = rmax <= 320 ? (int)(ceil_div(rmax, 32) * 32) : 256;
    const int64_t rtiles = ceil_div(rmax, T);
    static bool attr = false;
    if (!attr) {
      VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_gemv_n_cp<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    // splits: fill the resident slots once (>= 32 columns per CTA)
    const int64_t per = rtiles * a.nbatch;
    const size_t smem_est = ((size_t)S * T + ceil_div(cmax, 64)) * sizeof(cplx);
    int occ = 1;
    VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gemv_n_cp<S>, T, smem_est));
    occ = std::max(1, occ);
    int64_t nsl = std::max<int64_t>(1, std::min<int64_t>((int64_t)occ * sm_count() / per, cmax / 32));
    int ns = (int)std::min<int64_t>(nsl, max_splits);
    while (ns > 1 && (int64_t)a.nbatch * ns * rmax > partials_cap) --ns;
    const int64_t ncmax = ceil_div(cmax, ns);
    const size_t smem = ((size_t)S * T + ncmax) * sizeof(cplx);
    dim3 grid(ns, (unsigned)rtiles, a.nbatch);
    launch_pdl(k_gemv_n_cp<S>, grid, dim3(T), smem, st, a, partials, rmax);
    VSIE_CHECK_LAUNCH();
    launch_gemv_sum(a, partials, ns, rmax, st);
    return;
  }
}

void launch_sum3(const cplx* in, int64_t chi_stride, int64_t ld_in, int64_t rows, int k, cplx* out, int64_t ld_out,
                 bool conj_out, cudaStream_t st) {
  const int64_t n = rows * k;
  if (n <= 0) return;
  launch_pdl(k_sum3, dim3((unsigned)std::min<int64_t>(ceil_div(n, kThreads), 148 * 8)), dim3(kThreads), 0, st, in,
             chi_stride, ld_in, rows, k, out, ld_out, conj_out);
  VSIE_CHECK_LAUNCH();
}

void launch_gemv_t(const GemvT& a, cplx* partials, int64_t partials_cap, int max_splits, cudaStream_t st) {
  int64_t rmax = 0, cmax = 0;
  for (int b = 0; b < a.nbatch; ++b) {
    rmax = std::max(rmax, a.R[b]);
    cmax = std::max(cmax, a.C[b]);
  }
  if (cmax == 0) return;
  const int64_t ctiles = ceil_div(cmax, kColsPerCta);
  const int nz = a.sum_batch ? 1 : a.nbatch;
  // row splits: fill two waves of resident CTAs when a split keeps >= 128 rows
  const int64_t slots = (int64_t)sm_count() * gemv_occupancy((const void*)k_gemv_t, kThreads);
  int ns = a.sum_batch ? 1 : pick_splits(ctiles * nz, rmax, 128, max_splits, 2 * slots);
  while (ns > 1 && (int64_t)nz * ns * cmax > partials_cap) --ns;
  dim3 grid((unsigned)ctiles, ns, nz);
  launch_pdl(k_gemv_t, grid, dim3(kThreads), 0, st, a, partials, cmax);
  VSIE_CHECK_LAUNCH();
  if (ns > 1) {
    SumArgs sa{};
    sa.nbatch = nz;
    sa.conj_out = a.conj_out;
    for (int b = 0; b < nz; ++b) {
      sa.y[b] = a.y[b];
      sa.n[b] = a.C[b];
    }
    if (ns >= 16) {
      dim3 g2((unsigned)ceil_div(cmax, kThreads / 32), nz);
      launch_pdl(k_sum_partials_warp, g2, dim3(kThreads), 0, st, sa, (const cplx*)partials, ns, cmax);
    } else {
      dim3 g2((unsigned)ceil_div(cmax, kThreads), nz);
      launch_pdl(k_sum_partials, g2, dim3(kThreads), 0, st, sa, (const cplx*)partials, ns, cmax);
    }
    VSIE_CHECK_LAUNCH();
  }
}

template <class F>
void set_smem_attr_once(F* f, bool& done) {
  if (!done) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    done = true;
  }
}

// persistent G1-step grids: the resident CTAs of every SM over the batch
int64_t g1_ctas_per_chi(int nbatch, const void* fn, size_t smem, int threads) {
  int occ = 1;
  VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
  occ = std::max(1, occ);
  return std::max<int64_t>(1, (int64_t)sm_count() * occ / std::max(1, nbatch));
}

void launch_expand_g1(const ExpandArgs& a, cudaStream_t st) {
  int r1max = 0;
  for (int b = 0; b < a.nbatch; ++b) r1max = std::max(r1max, a.r1[b]);
  VSIE_REQUIRE(r1max <= 32, VSIE_ERR_ARG, "expand: r1 > 32 not supported");
  // DMMA k-steps for 4 KT values of k, exact DFMA for r1 % 4 == 1 more (r1 = 17: 4 + 1
  // instead of 5 padded k-steps, cfg 5 expansion 2.62 -> 2.53 ms per chi); with r1 % 4 == 2
  // (r1 = 10) the padded DMMA step measured faster than two DFMA columns (14.6 vs 15.4 us at
  // cfg 2), so only the remainder 1 takes the DFMA path
  // r1 % 4 == 2 (r1 = 10, 18): the concatenated real / imaginary k-step (2 DMMAs instead of 3)
  int KT = r1max / 4, REMK = r1max % 4;
  if (REMK > 2) {
    KT = (r1max + 3) / 4;
    REMK = 0;
  }
  const int mt = (a.n1 + 7) / 8;
  const size_t smem = ((size_t)mt * std::max(KT, 1) * 32 + (size_t)8 * mt * REMK) * sizeof(cplx);
  VSIE_REQUIRE(smem <= 200 * 1024, VSIE_ERR_ARG, "expand: n1 * r1 too large for shared memory");
#define VSIE_EXP(K, R)                                                                                     \
  if (KT == K && REMK == R) {                                                                              \
    static bool d = false;                                                                                 \
    set_smem_attr_once(k_expand_g1<K, R>, d);                                                              \
    dim3 grid((unsigned)std::min<int64_t>(ceil_div(a.ncol, kColsPerCtaG1),                                 \
                                          g1_ctas_per_chi(a.nbatch, (const void*)k_expand_g1<K, R>, smem, kG1Threads)), a.nbatch); \
    ExpandArgs ab = a;                                                                                     \
    const double rounds = (double)ceil_div(a.ncol, kColsPerWarp) / ((double)grid.x * kWarpsG1);            \
    ab.balanced = rounds >= 1.0 && rounds < 0.9 * std::ceil(rounds);                                       \
    launch_pdl(k_expand_g1<K, R>, grid, dim3(kG1Threads), smem, st, ab);                                   \
    VSIE_CHECK_LAUNCH();                                                                                   \
    return;                                                                                                \
  }
  VSIE_EXP(0, 1) VSIE_EXP(0, 2) VSIE_EXP(1, 0) VSIE_EXP(1, 1) VSIE_EXP(1, 2) VSIE_EXP(2, 0) VSIE_EXP(2, 1)
  VSIE_EXP(2, 2) VSIE_EXP(3, 0) VSIE_EXP(3, 1) VSIE_EXP(3, 2) VSIE_EXP(4, 0) VSIE_EXP(4, 1) VSIE_EXP(4, 2)
  VSIE_EXP(5, 0) VSIE_EXP(5, 1) VSIE_EXP(5, 2) VSIE_EXP(6, 0) VSIE_EXP(6, 1) VSIE_EXP(6, 2) VSIE_EXP(7, 0)
  VSIE_EXP(7, 1) VSIE_EXP(7, 2) VSIE_EXP(8, 0)
  VSIE_REQUIRE(false, VSIE_ERR_ARG, "expand: unsupported r1");
#undef VSIE_EXP
}

// the TMA-ring G1^T (single RHS: every chi's columns contiguous); false if the shape does
// not fit it (the caller then runs k_reduce_g1)
bool launch_reduce_g1_tma(const ReduceArgs& a, cudaStream_t st) {
  if (a.cols_per_rhs < a.ncol || a.ncol <= 0) return false;

  int r1max = 0;
  for (int b = 0; b < a.nbatch; ++b) r1max = std::max(r1max, a.r1[b]);
  if (r1max > 32) return false;
  int NT = r1max / 8, REM = r1max % 8;
  if (REM > 2) {
    NT = (r1max + 7) / 8;
    REM = 0;
  }
  const int n1 = a.n1, ks_n = (n1 + 3) / 4;
  // the upper half's partial sums (32 lanes x 6 NT + 2 REM doubles) fit in one tile of u
  if (32 * (6 * std::max(NT, 1) + 2 * std::max(REM, 1)) > 16 * n1) return false;
  const int64_t frag = 256 + ((int64_t)ks_n * std::max(NT, 1) * 32 + 4LL * ks_n * REM) * (int64_t)sizeof(cplx);
  const int64_t stage_off = (frag + 127) / 128 * 128;
  // two 8-column tiles per stage (a warp pair on each): cfg 4 (n1 = 200, 51 KB stages, 3 of
  // them) pair step 0.458 -> 0.438 ms although the kernel alone is ~5% slower -- its smaller
  // smem footprint lets the next kernel's CTAs become resident under its tail (PDL); one tile
  // per stage only when two would not leave three stages
  const int q = stage_off + 3LL * 16 * n1 * (int64_t)sizeof(cplx) <= 227 * 1024 ? 2 : 1;
  const int64_t stage_bytes = 8LL * q * n1 * (int64_t)sizeof(cplx);
  // CTAs per SM: one with as many stages as fit for long streams (cfg 4: 120 us vs 139 us for
  // two per SM with half the stages each), two when each CTA would get few stages (cfg 2:
  // ~17 stages per CTA, pair step 0.158 vs 0.170 ms: pipeline fill and drain dominate)
  const int64_t nst_all = ceil_div(a.ncol, 8LL * q);
  int cps_sm = nst_all / std::max(1, sm_count() / std::max(1, a.nbatch)) < 64 ? 2 : 1;
  int64_t smem_max = cps_sm == 1 ? 227 * 1024 : 233472 / 2 - 1024;
  int ns = (int)std::min<int64_t>(16, (smem_max - stage_off) / stage_bytes);
  if (ns < 3 && cps_sm == 2) {
    cps_sm = 1;
    smem_max = 227 * 1024;
    ns = (int)std::min<int64_t>(16, (smem_max - stage_off) / stage_bytes);
  }
  if (ns < 2) return false;
  const int ngroups = std::max(1, std::min(ns, kRtPairs / q));
  const size_t smem = (size_t)(stage_off + ns * stage_bytes);
  const int64_t nst = ceil_div(a.ncol, 8LL * q);
  dim3 grid((unsigned)std::min<int64_t>(nst, std::max(1, cps_sm * sm_count() / std::max(1, a.nbatch))), a.nbatch);
  const dim3 blk(32 * (2 * q * ngroups + 1));
#define VSIE_RT(K, R)                                                                                     \
  if (NT == K && REM == R) {                                                                              \
    static bool d0 = false, d1 = false;                                                                   \
    if (a.conj_u) {                                                                                       \
      if (!d1) {                                                                                          \
        VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_reduce_g1_tma<K, R, true>,                                 \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
        d1 = true;                                                                                        \
      }                                                                                                   \
      launch_pdl(k_reduce_g1_tma<K, R, true>, grid, blk, smem, st, a, q, ns, stage_off);     \
    } else {                                                                                              \
      if (!d0) {                                                                                          \
        VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_reduce_g1_tma<K, R, false>,                                \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
        d0 = true;                                                                                        \
      }                                                                                                   \
      launch_pdl(k_reduce_g1_tma<K, R, false>, grid, blk, smem, st, a, q, ns, stage_off);    \
    }                                                                                                     \
    VSIE_CHECK_LAUNCH();                                                                                  \
    return true;                                                                                          \
  }
  VSIE_RT(0, 1) VSIE_RT(0, 2) VSIE_RT(1, 0) VSIE_RT(1, 1) VSIE_RT(1, 2) VSIE_RT(2, 0) VSIE_RT(2, 1)
  VSIE_RT(2, 2) VSIE_RT(3, 0) VSIE_RT(3, 1) VSIE_RT(3, 2) VSIE_RT(4, 0)
#undef VSIE_RT
  return false;
}

void launch_reduce_g1(const ReduceArgs& a, cudaStream_t st, bool tma) {
  if (tma && launch_reduce_g1_tma(a, st)) return;
  int r1max = 0;
  for (int b = 0; b < a.nbatch; ++b) r1max = std::max(r1max, a.r1[b]);
  VSIE_REQUIRE(r1max <= 32, VSIE_ERR_ARG, "reduce: r1 > 32 not supported");
  // DMMA n-tiles for 8 NT values of a, exact DFMA for r1 % 8 <= 2 more
  int NT = r1max / 8, REM = r1max % 8;
  if (REM > 2) {
    NT = (r1max + 7) / 8;
    REM = 0;
  }
  const int ks_n = (a.n1 + 3) / 4;
  const size_t smem = ((size_t)ks_n * std::max(NT, 1) * 32 + (size_t)4 * ks_n * REM) * sizeof(cplx);
  VSIE_REQUIRE(smem <= 200 * 1024, VSIE_ERR_ARG, "reduce: n1 * r1 too large for shared memory");
#define VSIE_RED(K, R)                                                                                     \
  if (NT == K && REM == R) {                                                                               \
    static bool d = false;                                                                                 \
    set_smem_attr_once(k_reduce_g1<K, R>, d);                                                              \
    dim3 grid((unsigned)std::min<int64_t>(ceil_div(a.ncol, kColsPerWarp * kRedWarps),                      \
                                          g1_ctas_per_chi(a.nbatch, (const void*)k_reduce_g1<K, R>, smem, kRedThreads)), a.nbatch); \
    launch_pdl(k_reduce_g1<K, R>, grid, dim3(kRedThreads), smem, st, a);                                   \
    VSIE_CHECK_LAUNCH();                                                                                   \
    return;                                                                                                \
  }
  VSIE_RED(0, 1) VSIE_RED(0, 2) VSIE_RED(1, 0) VSIE_RED(1, 1) VSIE_RED(1, 2) VSIE_RED(2, 0) VSIE_RED(2, 1)
  VSIE_RED(2, 2) VSIE_RED(3, 0) VSIE_RED(3, 1) VSIE_RED(3, 2) VSIE_RED(4, 0)
  VSIE_REQUIRE(false, VSIE_ERR_ARG, "reduce: unsupported r1");
#undef VSIE_RED
}

}  // namespace vsie
