// TT-core contraction kernels of the Z_bc apply.
//
// Forward (Eq. 17), per chi:
//   y4 = G4 x            -> k_gemv_n   (r3 x m GEMV, HBM stream of G4)
//   Y3 = G3 y4           -> k_gemv_n   ((r2 n3) x r3 GEMV, HBM stream of G3)
//   Y2 = G2 Y3           -> zgemm      ((r1 n2) x r2 times r2 x n3)
//   y  = G1 Y2           -> k_expand_g1 (n1 x r1 times r1 x (n2 n3), coalesced voxel writes)
// Transpose (Eqs. 18-19), per chi, then summed over chi:
//   W1 = G1^T u          -> k_reduce_g1 (skinny reduction over i1, smem-staged)
//   W2 = G2^T W1         -> zgemm (T)
//   z3 = G3^T W2         -> k_gemv_t   (column dot products, deterministic split over rows)
//   z  = sum_chi G4^T z3 -> k_gemv_t   (sum_batch)
// All split reductions are deterministic: partials are summed in a fixed order
// by the last-arriving CTA (threadfence + ticket counter), so results are
// bitwise reproducible run to run.
#include "kernels.cuh"

#include <algorithm>

namespace vsie {

namespace {

constexpr int kThreads = 256;
constexpr int kXChunk = 512;

__device__ __forceinline__ cplx ldg_c(const cplx* p) { return __ldg(p); }

__global__ void __launch_bounds__(kThreads) k_gemv_n(GemvN a, cplx* __restrict__ partials,
                                                     unsigned* __restrict__ counters, int64_t rmax) {
  const int b = blockIdx.z;
  const int64_t R = a.R[b], C = a.C[b];
  const int64_t rt = blockIdx.y;
  if (rt * kThreads >= R) return;
  const int nsplit = gridDim.x, s = blockIdx.x;
  const int64_t c0 = C * s / nsplit, c1 = C * (s + 1) / nsplit;
  const int64_t row = rt * kThreads + threadIdx.x;
  const bool act = row < R;
  __shared__ cplx xs[kXChunk];
  cplx acc0 = cmk(0, 0), acc1 = acc0, acc2 = acc0, acc3 = acc0;
  const cplx* __restrict__ X = a.x[b];
  const cplx* __restrict__ A = a.A[b];
  for (int64_t cc = c0; cc < c1; cc += kXChunk) {
    const int len = (int)min((int64_t)kXChunk, c1 - cc);
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += kThreads) xs[j] = ldg_c(X + cc + j);
    __syncthreads();
    if (act) {
      const cplx* Ap = A + row + R * cc;
      int j = 0;
      for (; j + 4 <= len; j += 4) {
        const cplx v0 = ldg_c(Ap + R * j), v1 = ldg_c(Ap + R * (j + 1));
        const cplx v2 = ldg_c(Ap + R * (j + 2)), v3 = ldg_c(Ap + R * (j + 3));
        cfma(acc0, v0, xs[j]);
        cfma(acc1, v1, xs[j + 1]);
        cfma(acc2, v2, xs[j + 2]);
        cfma(acc3, v3, xs[j + 3]);
      }
      for (; j < len; ++j) cfma(acc0, ldg_c(Ap + R * j), xs[j]);
    }
  }
  const cplx sum = cadd(cadd(acc0, acc1), cadd(acc2, acc3));
  if (nsplit == 1) {
    if (act) a.y[b][row] = sum;
    return;
  }
  if (act) partials[((int64_t)b * nsplit + s) * rmax + row] = sum;
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  unsigned* ctr = counters + (int64_t)b * gridDim.y + rt;
  if (threadIdx.x == 0) last = (atomicAdd(ctr, 1u) == (unsigned)(nsplit - 1));
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (act) {
    cplx tot = cmk(0, 0);
    for (int q = 0; q < nsplit; ++q) tot = cadd(tot, __ldcg(partials + ((int64_t)b * nsplit + q) * rmax + row));
    a.y[b][row] = tot;
  }
  if (threadIdx.x == 0) *ctr = 0;
}

constexpr int kWarps = kThreads / 32;
constexpr int kCPW = 4;                     // columns per warp
constexpr int kColsPerCta = kWarps * kCPW;  // 32

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y[c] = sum_r A[r + R c] x[r]  over rows [r0, r1) of this split.
__global__ void __launch_bounds__(kThreads) k_gemv_t(GemvT a, cplx* __restrict__ partials,
                                                     unsigned* __restrict__ counters, int64_t cmax) {
  const bool conj_out = a.conj_out;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ct = blockIdx.x;
  const int nsplit = gridDim.y, s = blockIdx.y;
  const int bz = blockIdx.z;
  const int nb = a.sum_batch ? a.nbatch : 1;
  // in sum_batch mode all batches share the output columns (same C)
  const int64_t Cout = a.C[a.sum_batch ? 0 : bz];
  if ((int64_t)ct * kColsPerCta >= Cout) return;
  const int64_t cbase = (int64_t)ct * kColsPerCta + warp * kCPW;
  cplx acc[kCPW];
#pragma unroll
  for (int j = 0; j < kCPW; ++j) acc[j] = cmk(0, 0);
  for (int bb = 0; bb < nb; ++bb) {
    const int b = a.sum_batch ? bb : bz;
    const int64_t R = a.R[b];
    const int64_t r0 = R * s / nsplit, r1 = R * (s + 1) / nsplit;
    const cplx* __restrict__ A = a.A[b];
    const cplx* __restrict__ X = a.x[b];
    for (int64_t r = r0 + lane; r < r1; r += 32) {
      const cplx xv = ldg_c(X + r);
#pragma unroll
      for (int j = 0; j < kCPW; ++j) {
        const int64_t c = cbase + j;
        if (c < Cout) cfma(acc[j], ldg_c(A + r + R * c), xv);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kCPW; ++j) {
    acc[j].x = warp_sum(acc[j].x);
    acc[j].y = warp_sum(acc[j].y);
  }
  if (nsplit == 1) {
    if (lane < kCPW) {
      cplx v = acc[0];
#pragma unroll
      for (int j = 1; j < kCPW; ++j)
        if (lane == j) v = acc[j];
      const int64_t c = cbase + lane;
      if (c < Cout) a.y[bz][c] = conj_out ? cconj(v) : v;
    }
    return;
  }
  if (lane < kCPW) {
    cplx v = acc[0];
#pragma unroll
    for (int j = 1; j < kCPW; ++j)
      if (lane == j) v = acc[j];
    const int64_t c = cbase + lane;
    if (c < Cout) partials[((int64_t)bz * nsplit + s) * cmax + c] = v;
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  unsigned* ctr = counters + (int64_t)bz * gridDim.x + ct;
  if (threadIdx.x == 0) last = (atomicAdd(ctr, 1u) == (unsigned)(nsplit - 1));
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int t = threadIdx.x; t < kColsPerCta; t += kThreads) {
    const int64_t c = (int64_t)ct * kColsPerCta + t;
    if (c < Cout) {
      cplx tot = cmk(0, 0);
      for (int q = 0; q < nsplit; ++q) tot = cadd(tot, __ldcg(partials + ((int64_t)bz * nsplit + q) * cmax + c));
      a.y[bz][c] = conj_out ? cconj(tot) : tot;
    }
  }
  if (threadIdx.x == 0) *ctr = 0;
}

// ----------------------------------------------------------------------------- G1 expansion
constexpr int kExpCols = 64;
constexpr int kExpGroup = 8;

__global__ void __launch_bounds__(kThreads) k_expand_g1(ExpandArgs a) {
  const int b = blockIdx.y;
  const int n1 = a.n1, r1 = a.r1[b];
  const int64_t col0 = (int64_t)blockIdx.x * kExpCols;
  if (col0 >= a.ncol) return;
  const int ncols = (int)min((int64_t)kExpCols, a.ncol - col0);
  extern __shared__ cplx sm[];
  cplx* G1s = sm;             // [a1][i1] = G1 column-major
  cplx* Y2s = sm + n1 * r1;   // [c][a1]
  const cplx* __restrict__ G1 = a.G1[b];
  for (int t = threadIdx.x; t < n1 * r1; t += kThreads) G1s[t] = ldg_c(G1 + t);
  const cplx* __restrict__ Y2 = a.Y2[b] + (int64_t)r1 * col0;
  for (int t = threadIdx.x; t < r1 * ncols; t += kThreads) Y2s[t] = ldg_c(Y2 + t);
  __syncthreads();
  const int ngroups = (ncols + kExpGroup - 1) / kExpGroup;
  cplx* __restrict__ Y = a.y[b];
  for (int f = threadIdx.x; f < n1 * ngroups; f += kThreads) {
    const int i1 = f % n1, gi = f / n1;
    cplx acc[kExpGroup];
#pragma unroll
    for (int j = 0; j < kExpGroup; ++j) acc[j] = cmk(0, 0);
    const cplx* yb = Y2s + r1 * (gi * kExpGroup);
    for (int a1 = 0; a1 < r1; ++a1) {
      const cplx gv = G1s[i1 + n1 * a1];
#pragma unroll
      for (int j = 0; j < kExpGroup; ++j) cfma(acc[j], gv, yb[a1 + r1 * j]);
    }
#pragma unroll
    for (int j = 0; j < kExpGroup; ++j) {
      const int cl = gi * kExpGroup + j;
      if (cl < ncols) {
        const int64_t c = col0 + cl;
        const int64_t rhs = c / a.cols_per_rhs, cc = c - rhs * a.cols_per_rhs;
        Y[rhs * a.ld_rhs + cc * n1 + i1] = acc[j];
      }
    }
  }
}

// ----------------------------------------------------------------------------- G1^T reduction
constexpr int kRedCols = 64;
constexpr int kRedK = 32;
constexpr int kRedGroups = kThreads / kRedCols;  // 4 a1-groups
constexpr int kRedMaxAcc = 8;                    // r1 <= 32 per pass

__global__ void __launch_bounds__(kThreads) k_reduce_g1(ReduceArgs a) {
  const int b = blockIdx.y;
  const int n1 = a.n1, r1 = a.r1[b];
  const int64_t col0 = (int64_t)blockIdx.x * kRedCols;
  if (col0 >= a.ncol) return;
  const int ncols = (int)min((int64_t)kRedCols, a.ncol - col0);
  __shared__ cplx us[kRedK][kRedCols + 1];
  extern __shared__ cplx G1s[];  // [a1][i1] = G1 column-major, n1 * r1
  const cplx* __restrict__ G1 = a.G1[b];
  for (int t = threadIdx.x; t < n1 * r1; t += kThreads) G1s[t] = ldg_c(G1 + t);
  const int c = threadIdx.x % kRedCols, ag = threadIdx.x / kRedCols;
  const cplx* __restrict__ U = a.u[b];
  for (int abase = 0; abase < r1; abase += kRedGroups * kRedMaxAcc) {
    cplx acc[kRedMaxAcc];
#pragma unroll
    for (int j = 0; j < kRedMaxAcc; ++j) acc[j] = cmk(0, 0);
    for (int k0 = 0; k0 < n1; k0 += kRedK) {
      const int klen = min(kRedK, n1 - k0);
      __syncthreads();
      // stage u[k0:k0+klen, col0:col0+ncols] transposed as us[i1][c]
      for (int t = threadIdx.x; t < kRedK * kRedCols; t += kThreads) {
        const int kk = t % kRedK, cl = t / kRedK;
        cplx v = cmk(0, 0);
        if (kk < klen && cl < ncols) {
          const int64_t cg = col0 + cl;
          const int64_t rhs = cg / a.cols_per_rhs, cc = cg - rhs * a.cols_per_rhs;
          v = ldg_c(U + rhs * a.ld_rhs + cc * n1 + k0 + kk);
          if (a.conj_u) v.y = -v.y;
        }
        us[kk][cl] = v;
      }
      __syncthreads();
      for (int kk = 0; kk < klen; ++kk) {
        const cplx uv = us[kk][c];
#pragma unroll
        for (int j = 0; j < kRedMaxAcc; ++j) {
          const int a1 = abase + ag + kRedGroups * j;
          if (a1 < r1) cfma(acc[j], G1s[k0 + kk + n1 * a1], uv);
        }
      }
    }
    if (c < ncols) {
      cplx* W = a.W1[b] + (int64_t)r1 * (col0 + c);
#pragma unroll
      for (int j = 0; j < kRedMaxAcc; ++j) {
        const int a1 = abase + ag + kRedGroups * j;
        if (a1 < r1) W[a1] = acc[j];
      }
    }
  }
}

int pick_splits(int64_t other_ctas, int64_t len, int min_len, int max_splits) {
  const int64_t target = 148 * 6;
  int64_t s = target / std::max<int64_t>(1, other_ctas);
  s = std::min<int64_t>(s, len / std::max(1, min_len));
  s = std::min<int64_t>(s, max_splits);
  return (int)std::max<int64_t>(1, s);
}

}  // namespace

void launch_gemv_n(const GemvN& a, cplx* partials, unsigned* counters, int max_splits, cudaStream_t st) {
  int64_t rmax = 0, cmax = 0;
  for (int b = 0; b < a.nbatch; ++b) {
    rmax = std::max(rmax, a.R[b]);
    cmax = std::max(cmax, a.C[b]);
  }
  if (rmax == 0) return;
  const int64_t rtiles = ceil_div(rmax, kThreads);
  const int ns = pick_splits(rtiles * a.nbatch, cmax, 32, max_splits);
  dim3 grid(ns, (unsigned)rtiles, a.nbatch);
  k_gemv_n<<<grid, kThreads, 0, st>>>(a, partials, counters, rmax);
  VSIE_CHECK_LAUNCH();
}

void launch_gemv_t(const GemvT& a, cplx* partials, unsigned* counters, int max_splits, cudaStream_t st) {
  int64_t rmax = 0, cmax = 0;
  for (int b = 0; b < a.nbatch; ++b) {
    rmax = std::max(rmax, a.R[b]);
    cmax = std::max(cmax, a.C[b]);
  }
  if (cmax == 0) return;
  const int64_t ctiles = ceil_div(cmax, kColsPerCta);
  const int nz = a.sum_batch ? 1 : a.nbatch;
  const int ns = a.sum_batch ? 1 : pick_splits(ctiles * nz, rmax, 256, max_splits);
  dim3 grid((unsigned)ctiles, ns, nz);
  k_gemv_t<<<grid, kThreads, 0, st>>>(a, partials, counters, cmax);
  VSIE_CHECK_LAUNCH();
}

void launch_expand_g1(const ExpandArgs& a, cudaStream_t st) {
  int r1max = 0;
  for (int b = 0; b < a.nbatch; ++b) r1max = std::max(r1max, a.r1[b]);
  const size_t smem = (size_t)(a.n1 * r1max + r1max * kExpCols) * sizeof(cplx);
  VSIE_REQUIRE(smem <= 220 * 1024, VSIE_ERR_ARG, "expand: n1 * r1 too large for shared memory");
  static bool configured = false;
  if (!configured) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_expand_g1, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    configured = true;
  }
  dim3 grid((unsigned)ceil_div(a.ncol, kExpCols), a.nbatch);
  k_expand_g1<<<grid, kThreads, smem, st>>>(a);
  VSIE_CHECK_LAUNCH();
}

void launch_reduce_g1(const ReduceArgs& a, cudaStream_t st) {
  int r1max = 0;
  for (int b = 0; b < a.nbatch; ++b) r1max = std::max(r1max, a.r1[b]);
  const size_t smem = (size_t)a.n1 * r1max * sizeof(cplx);
  VSIE_REQUIRE(smem + sizeof(cplx) * kRedK * (kRedCols + 1) <= 220 * 1024, VSIE_ERR_ARG,
               "reduce: n1 * r1 too large for shared memory");
  static bool configured = false;
  if (!configured) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_reduce_g1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024 - (int)(sizeof(cplx) * kRedK * (kRedCols + 1))));
    configured = true;
  }
  dim3 grid((unsigned)ceil_div(a.ncol, kRedCols), a.nbatch);
  k_reduce_g1<<<grid, kThreads, smem, st>>>(a);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
