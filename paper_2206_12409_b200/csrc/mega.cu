// Persistent dataflow apply (see mega.cuh for the design).  Tile types:
//   TN   y[r] = sum_c A[r + ld c] x[c] over a <= 128-row block   (G4 x, G3 y4)
//   TT   z[c] = sum_r A[r + ld c] v[r] over a row range          (G3^T W2, G4^T z3)
//   GEMM 64 x 32 complex tile on FP64 tensor cores (DMMA)       (G2 Y3, G2^T W1)
//   EXP  y = G1 Y2 over 256 voxel columns (DMMA)                 (forward G1 step)
//   RED  W1 = G1^T u over 256 voxel columns (DMMA)               (transpose G1 step)
#include "mega.cuh"
#include "dmma_tile.cuh"

#include <algorithm>
#include <cstdlib>

namespace vsie {

namespace {

constexpr int MT = 256;    // threads per CTA
#ifndef MEGA_MIN_BLOCKS
#define MEGA_MIN_BLOCKS 2
#endif
constexpr int NWARP = MT / 32;
constexpr int kRowsTN = 32;    // TN row block (one row per lane, deep column pipeline)
constexpr int kRowsRange = 1024; // TN2 row range of G4 x (partials stride)
constexpr int kGrp = 16;         // first-level group of the G4 x split reduction
constexpr int kRowsTT = 1024;  // TT row range of the G3 transpose
constexpr int kColsTile = 256; // EXP / RED columns per tile
// GEMM tiles (dmma_tile.cuh): forward (4 x 2 warps) = 64 x 32, transpose (2 x 4) = 32 x 64
using tc::FWA; using tc::FWB; using tc::AWA; using tc::AWB;
using tc::FTM; using tc::FTN; using tc::ATM; using tc::ATN; using tc::GKC;
using tc::GemmSmem; using tc::gemm_tile;

// ------------------------------------------------------------------ sync primitives
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// block-wide wait until flag == epoch.  A dependency that never arrives is a bug, not a
// state to wait out: after 4 s the kernel traps (launch error) instead of hanging the GPU.
// block-wide wait for the contiguous flags f[0..n): one thread per flag, in parallel
__device__ __noinline__ void wait_flags(const unsigned* f, int n, unsigned epoch, unsigned long long* t_ready) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned ns = 32;
    uint64_t t0 = 0;
    while (ld_acquire(f + i) != epoch) {
      __nanosleep(ns);
      ns = min(ns * 2, 256u);
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
  __syncthreads();
  if (t_ready && threadIdx.x == 0) *t_ready = globaltimer_ns();
}
__device__ __forceinline__ void wait_flag(const unsigned* f, unsigned epoch, unsigned long long* t_ready = nullptr) {
  if (threadIdx.x == 0) {
    unsigned ns = 32;
    uint64_t t0 = 0;
    while (ld_acquire(f) != epoch) {
      __nanosleep(ns);
      ns = min(ns * 2, 256u);
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
    if (t_ready) *t_ready = globaltimer_ns();
  }
  __syncthreads();
}
// all threads wrote their part of a group partial; returns true in every thread of
// the CTA that arrived last (n arrivals), after which the partials of the group are
// visible to it
__device__ __forceinline__ bool arrive_last(unsigned* ticket, unsigned n, int* s_flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket, 1u);
    *s_flag = (t == n - 1);
    if (t == n - 1) *ticket = 0;   // self-reset for the next launch
  }
  __syncthreads();
  const bool last = *s_flag != 0;
  if (last) __threadfence();
  return last;
}
// count one finished unit of a group of n; the unit completing the group publishes flag
__device__ __forceinline__ void count_and_publish(unsigned* cnt, unsigned n, unsigned* flag, unsigned epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(cnt, 1u);
    if (t == n - 1) {
      *cnt = 0;
      __threadfence();
      st_release(flag, epoch);
    }
  }
}
__device__ __forceinline__ void publish(unsigned* flag, unsigned epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(flag, epoch);
}

__device__ __forceinline__ cplx ld_stream(const cplx* p) {
  cplx v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ cplx ld_cg(const cplx* p) { return __ldcg(p); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__host__ __device__ __forceinline__ int64_t blo(int64_t n, int64_t k, int64_t i) { return n * i / k; }
// index of the balanced block (n items in k blocks) containing item r
__device__ __forceinline__ int64_t block_of(int64_t n, int64_t k, int64_t r) {
  int64_t b = (r * k) / n;
  while (b + 1 < k && blo(n, k, b + 1) <= r) ++b;
  while (b > 0 && blo(n, k, b) > r) --b;
  return b;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void zmma(double (&cr)[2], double (&ci)[2], cplx a, cplx b) {
  dmma(cr[0], cr[1], a.x, b.x);
  dmma(cr[0], cr[1], -a.y, b.y);
  dmma(ci[0], ci[1], a.x, b.y);
  dmma(ci[0], ci[1], a.y, b.x);
}

// ------------------------------------------------------------------ TN: row block GEMV
// acc over columns [c0, c1) of rows [r0, r0 + nr), nr <= 128: warp w takes columns
// c0 + w + 8 j, lane l rows l + 32 q; two columns per pipeline step, the next step's
// loads in flight while this one is consumed.  Result (fixed-order sum over warps) in
// red[0][0..nr).
template <int NQ>
__device__ __noinline__ void tn_block(const cplx* __restrict__ A, int64_t ld, int64_t r0, int nr, int64_t c0, int64_t c1,
                         const cplx* __restrict__ x, cplx (*red)[kRowsTN]) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const cplx* p[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int row = l + 32 * q;
    p[q] = A + r0 + (row < nr ? row : 0);
  }
  cplx acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = cmk(0, 0);
  // CPS columns (c, c + 8, ...) per pipeline step; the next step's CPS NQ loads are
  // issued before this step's are consumed (2 CPS NQ = 8..16 streaming loads in flight)
  constexpr int CPS = NQ == 1 ? 8 : (NQ == 2 ? 4 : 2);
  int64_t c = c0 + w;
  if (c + 8 * (CPS - 1) < c1) {
    cplx v[CPS][NQ], xv[CPS];
#pragma unroll
    for (int j = 0; j < CPS; ++j) {
      xv[j] = x[c + 8 * j];
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[j][q] = ld_stream(p[q] + ld * (c + 8 * j));
    }
    c += 8 * CPS;
    for (; c + 8 * (CPS - 1) < c1; c += 8 * CPS) {
      cplx wv[CPS][NQ], xw[CPS];
#pragma unroll
      for (int j = 0; j < CPS; ++j) {
        xw[j] = x[c + 8 * j];
#pragma unroll
        for (int q = 0; q < NQ; ++q) wv[j][q] = ld_stream(p[q] + ld * (c + 8 * j));
      }
#pragma unroll
      for (int j = 0; j < CPS; ++j)
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          cfma(acc[q], v[j][q], xv[j]);
          v[j][q] = wv[j][q];
        }
#pragma unroll
      for (int j = 0; j < CPS; ++j) xv[j] = xw[j];
    }
#pragma unroll
    for (int j = 0; j < CPS; ++j)
#pragma unroll
      for (int q = 0; q < NQ; ++q) cfma(acc[q], v[j][q], xv[j]);
  }
  for (; c < c1; c += 8) {
    const cplx xs = x[c];
#pragma unroll
    for (int q = 0; q < NQ; ++q) cfma(acc[q], ld_stream(p[q] + ld * c), xs);
  }
  __syncthreads();  // red may still be read by a previous tile's epilogue
#pragma unroll
  for (int q = 0; q < NQ; ++q) red[w][l + 32 * q] = acc[q];
  __syncthreads();
  if (threadIdx.x < nr) {
    cplx s = red[0][threadIdx.x];
#pragma unroll
    for (int ww = 1; ww < NWARP; ++ww) s = cadd(s, red[ww][threadIdx.x]);
    red[0][threadIdx.x] = s;   // only this thread reads / writes column threadIdx.x
  }
  __syncthreads();
}

__device__ void tn_dispatch(const cplx* A, int64_t ld, int64_t r0, int nr, int64_t c0, int64_t c1, const cplx* x,
                            cplx (*red)[kRowsTN], cplx* xs) {
  // x[c0, c1) (<= 2048 values, produced in-launch for G3) staged once per tile in smem
  __syncthreads();
  for (int64_t c = c0 + threadIdx.x; c < c1; c += MT) xs[c - c0] = ld_cg(x + c);
  __syncthreads();
  x = xs - c0;
  const int nq = (nr + 31) / 32;
  if (nq <= 1) tn_block<1>(A, ld, r0, nr, c0, c1, x, red);
  else if (nq == 2) tn_block<2>(A, ld, r0, nr, c0, c1, x, red);
  else if (nq == 3) tn_block<3>(A, ld, r0, nr, c0, c1, x, red);
  else tn_block<4>(A, ld, r0, nr, c0, c1, x, red);
}

// ------------------------------------------------------------------ TN2: row range x column split
// out[r] = sum_{c in [c0, c1)} A[row0 + r + ld c] xs[c - c0], r < nrows <= 1024: thread t owns
// rows t + 256 q (q < RPT); every column of the tile is read by the whole CTA as one
// contiguous segment of nrows elements (whole DRAM pages).  CPS columns per pipeline step,
// the next step's loads in flight while this one is consumed; x comes from smem.
template <int RPT>
__device__ __noinline__ void tn2_tile(const cplx* __restrict__ A, int64_t ld, int64_t row0, int nrows, int64_t c0,
                                      int64_t c1, const cplx* xs, cplx* __restrict__ out) {
  constexpr int CPS = RPT == 1 ? 8 : (RPT == 2 ? 6 : (RPT == 3 ? 3 : 2));
  const int t = threadIdx.x;
  const cplx* p[RPT];
  bool act[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = t + MT * q;
    act[q] = r < nrows;
    p[q] = A + row0 + (act[q] ? r : nrows - 1);
  }
  cplx acc[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) acc[q] = cmk(0, 0);
  int64_t c = c0;
  if (c + CPS <= c1) {
    cplx v[CPS][RPT];
#pragma unroll
    for (int j = 0; j < CPS; ++j)
#pragma unroll
      for (int q = 0; q < RPT; ++q) v[j][q] = act[q] ? ld_stream(p[q] + ld * (c + j)) : cmk(0, 0);
    c += CPS;
    for (; c + CPS <= c1; c += CPS) {
      cplx w[CPS][RPT];
#pragma unroll
      for (int j = 0; j < CPS; ++j)
#pragma unroll
        for (int q = 0; q < RPT; ++q) w[j][q] = act[q] ? ld_stream(p[q] + ld * (c + j)) : cmk(0, 0);
#pragma unroll
      for (int j = 0; j < CPS; ++j) {
        const cplx xv = xs[c - CPS + j - c0];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          cfma(acc[q], v[j][q], xv);
          v[j][q] = w[j][q];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CPS; ++j) {
      const cplx xv = xs[c - CPS + j - c0];
#pragma unroll
      for (int q = 0; q < RPT; ++q) cfma(acc[q], v[j][q], xv);
    }
  }
  for (; c < c1; ++c) {
    const cplx xv = xs[c - c0];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (act[q]) cfma(acc[q], ld_stream(p[q] + ld * c), xv);
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q)
    if (act[q]) out[t + MT * q] = acc[q];
}

// stage x[c0, c1) in smem, then the TN2 tile (RPT from nrows)
__device__ void tn2_dispatch(const cplx* A, int64_t ld, int64_t row0, int nrows, int64_t c0, int64_t c1, const cplx* x,
                             cplx* xs, cplx* out) {
  __syncthreads();
  for (int64_t c = c0 + threadIdx.x; c < c1; c += MT) xs[c - c0] = ld_cg(x + c);
  __syncthreads();
  const int rpt = (nrows + MT - 1) / MT;
  if (rpt <= 1) tn2_tile<1>(A, ld, row0, nrows, c0, c1, xs, out);
  else if (rpt == 2) tn2_tile<2>(A, ld, row0, nrows, c0, c1, xs, out);
  else if (rpt == 3) tn2_tile<3>(A, ld, row0, nrows, c0, c1, xs, out);
  else tn2_tile<4>(A, ld, row0, nrows, c0, c1, xs, out);
}

// ------------------------------------------------------------------ TT: column dot products
// out[j] = sum_{r < nrows} A[row0 + r + ld (col0 + j)] vs[r], j < ncols (results in smem
// res[]).  Warp per column pair, lanes over rows in groups of 128 (4 loads per column),
// flattened (pair, group) steps software-pipelined; vs zero-padded to a multiple of 128.
__device__ __noinline__ void tt_cols(const cplx* __restrict__ A, int64_t ld, int64_t row0, int nrows, int64_t col0,
                                     int ncols, const cplx* vs, cplx* res) {
  // warp per group of CW columns, lanes over rows in groups of 128 (4 loads per column):
  // 4 CW streaming loads per step, the next row group's loads issued before this one's
  // are consumed; rows past nrows re-read the last row (their vs entries are zero)
  constexpr int CW = 3;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int ng = (nrows + 127) / 128;
  for (int gb = CW * w; gb < ncols; gb += CW * NWARP) {
    const cplx* col[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) col[j] = A + row0 + ld * (col0 + min(gb + j, ncols - 1));
    int roff[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) roff[u] = min(32 * u + l, nrows - 1);
    cplx buf[4][CW];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < CW; ++j) buf[u][j] = ld_stream(col[j] + roff[u]);
    cplx acc[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) acc[j] = cmk(0, 0);
    for (int g = 0; g < ng; ++g) {
      cplx nb[4][CW];
      if (g + 1 < ng) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = min((g + 1) * 128 + 32 * u + l, nrows - 1);
#pragma unroll
          for (int j = 0; j < CW; ++j) nb[u][j] = ld_stream(col[j] + r);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const cplx v = vs[g * 128 + 32 * u + l];
#pragma unroll
        for (int j = 0; j < CW; ++j) cfma(acc[j], buf[u][j], v);
      }
      if (g + 1 < ng) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < CW; ++j) buf[u][j] = nb[u][j];
      }
    }
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      acc[j].x = warp_sum(acc[j].x);
      acc[j].y = warp_sum(acc[j].y);
    }
    if (l == 0) {
#pragma unroll
      for (int j = 0; j < CW; ++j)
        if (gb + j < ncols) res[gb + j] = acc[j];
    }
  }
}

// ------------------------------------------------------------------ EXP: y = G1 Y2 on DMMA
// G1 fragments Af[(mtile * KT + ks) * 32 + lane] (A[g][t] of m8n8k4) staged per tile;
// warp task = 8 voxel columns; Y2 fragments read coherently (produced in-launch).
template <int KT>
__device__ __noinline__ void exp_tile(const cplx* __restrict__ G1, int n1, int r1, const cplx* __restrict__ Y2, int64_t c0,
                         int64_t c1, cplx* __restrict__ y, cplx* Af) {
  const int mt = (n1 + 7) / 8;
  __syncthreads();
  for (int e = threadIdx.x; e < mt * KT * 32; e += MT) {
    const int lane = e % 32, ks = (e / 32) % KT, m = e / (32 * KT);
    const int i1 = 8 * m + (lane >> 2), k = 4 * ks + (lane & 3);
    Af[e] = (i1 < n1 && k < r1) ? __ldg(G1 + i1 + (int64_t)n1 * k) : cmk(0, 0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  for (int64_t cb = c0 + 8 * warp; cb < c1; cb += 8 * NWARP) {
    cplx bf[KT];
    const int64_t cg = cb + g;
#pragma unroll
    for (int ks = 0; ks < KT; ++ks) {
      const int k = 4 * ks + t;
      bf[ks] = (cg < c1 && k < r1) ? ld_cg(Y2 + (int64_t)r1 * cg + k) : cmk(0, 0);
    }
    bool ok[2];
    cplx* out[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t c = cb + 2 * t + j;
      ok[j] = c < c1;
      out[j] = y + (ok[j] ? c : c0) * n1;
    }
    double bsum[KT];
#pragma unroll
    for (int ks = 0; ks < KT; ++ks) bsum[ks] = bf[ks].x + bf[ks].y;
    for (int m = 0; m < mt; ++m) {
      // 3 real DMMAs per complex product: P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi)
      double p1[2] = {0, 0}, p2[2] = {0, 0}, p3[2] = {0, 0};
#pragma unroll
      for (int ks = 0; ks < KT; ++ks) {
        const cplx av = Af[(m * KT + ks) * 32 + lane];
        dmma(p1[0], p1[1], av.x, bf[ks].x);
        dmma(p2[0], p2[1], av.y, bf[ks].y);
        dmma(p3[0], p3[1], av.x + av.y, bsum[ks]);
      }
      const int i1 = 8 * m + g;
      if (i1 < n1) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (ok[j]) __stcs(out[j] + i1, cmk(p1[j] - p2[j], p3[j] - p1[j] - p2[j]));
      }
    }
  }
}

// ------------------------------------------------------------------ RED: W1 = G1^T u on DMMA
template <int NT>
__device__ __noinline__ void red_tile(const cplx* __restrict__ G1, int n1, int r1, const cplx* __restrict__ u, bool conj_u,
                         int64_t c0, int64_t c1, cplx* __restrict__ W1, cplx* Bf) {
  const int ks_n = (n1 + 3) / 4;
  __syncthreads();
  for (int e = threadIdx.x; e < ks_n * NT * 32; e += MT) {
    const int lane = e % 32, nt = (e / 32) % NT, ks = e / (32 * NT);
    const int k = 4 * ks + (lane & 3), n = 8 * nt + (lane >> 2);
    Bf[e] = (k < n1 && n < r1) ? __ldg(G1 + k + (int64_t)n1 * n) : cmk(0, 0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const double sgn = conj_u ? -1.0 : 1.0;
  for (int64_t cb = c0 + 8 * warp; cb < c1; cb += 8 * NWARP) {
    const int64_t cg = cb + g;
    const bool cok = cg < c1;
    const cplx* __restrict__ U = u + (cok ? cg : c0) * n1;
    // 3 real DMMAs per complex product (see gemm_tile)
    double p1[NT][2], p2[NT][2], p3[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) p1[nt][0] = p1[nt][1] = p2[nt][0] = p2[nt][1] = p3[nt][0] = p3[nt][1] = 0;
    constexpr int UNR = 8;    // 8 k-steps (32 voxels of the column) in flight per lane
    for (int ks = 0; ks < ks_n; ks += UNR) {
      cplx av[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int k = 4 * (ks + q) + t;
        av[q] = ld_stream(U + (k < n1 ? k : n1 - 1));
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        if (ks + q < ks_n) {
          const int k = 4 * (ks + q) + t;
          const double ar = k < n1 ? av[q].x : 0.0, ai = k < n1 ? sgn * av[q].y : 0.0;
          const double as = ar + ai;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const cplx bv = Bf[((ks + q) * NT + nt) * 32 + lane];
            dmma(p1[nt][0], p1[nt][1], ar, bv.x);
            dmma(p2[nt][0], p2[nt][1], ai, bv.y);
            dmma(p3[nt][0], p3[nt][1], as, bv.x + bv.y);
          }
        }
      }
    }
    if (cok) {
      cplx* __restrict__ W = W1 + (int64_t)r1 * cg;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int aa = 8 * nt + 2 * t + j;
          if (aa < r1) W[aa] = cmk(p1[nt][j] - p2[nt][j], p3[nt][j] - p1[nt][j] - p2[nt][j]);
        }
    }
  }
}

// ------------------------------------------------------------------ shared memory of the kernel
struct MegaSmem {
  union {
    struct {
      cplx red[NWARP][kRowsTN];        // TN warp partials
      cplx xs[2048];                   // TN x staging (the tile's column range)
    } tn;
    GemmSmem gemm;                     // GEMM
    struct {
      cplx vs[2048];                   // TT vector (<= 2048 rows)
      cplx res[64];                    // TT column results
    } tt;
  } u;
  int flag;
  unsigned long long t_ready;   // diagnostics: when the tile's dependencies were satisfied
};

struct Q {  // tile coordinates
  int phase, chi;
  int64_t i;
};

__device__ __forceinline__ Q decode(const MegaPlan& p, int64_t t) {
  int s = 0;
  while (s + 1 < p.nseg && p.seg_off[s + 1] <= t) ++s;
  return Q{p.seg_phase[s], p.seg_chi[s], t - p.seg_off[s]};
}

// ------------------------------------------------------------------ forward tiles
__device__ __noinline__ void fwd_tile(const MegaArgs& a, const Q q, unsigned E, MegaSmem& sm, cplx* dyn) {
  const MegaPlan& p = a.p;
  const int c = q.chi;
  const MegaChi& ch = a.c[c];
  unsigned* S = a.sync;
  if (q.phase == 0) {
    // ---- y4 = G4 x: row range rr (<= 1024 rows) x column split s; two-level ticketed
    //      sum over the splits (groups of kGrp, then the groups), fixed order
    const int S4 = p.s4[c], nrr = p.nrb4[c];
    const int rr = (int)(q.i / S4), s = (int)(q.i % S4);
    const int64_t r0 = blo(ch.r3, nrr, rr), r1 = blo(ch.r3, nrr, rr + 1);
    const int nr = (int)(r1 - r0);
    const int64_t c0 = blo(a.mloc, S4, s), c1 = blo(a.mloc, S4, s + 1);
    const int ngrp = (S4 + kGrp - 1) / kGrp, grp = s / kGrp, gsz = min(kGrp, S4 - grp * kGrp);
    cplx* part = a.part + p.p_a[c] + (int64_t)rr * (S4 + ngrp) * kRowsRange;
    tn2_dispatch(ch.G4, ch.r3, r0, nr, c0, c1, a.x, sm.u.tn.xs, part + (int64_t)s * kRowsRange);
    if (arrive_last(S + p.o_tick_a[c] + rr * (ngrp + 1) + grp, gsz, &sm.flag)) {
      cplx* gpart = part + (int64_t)(S4 + grp) * kRowsRange;
      for (int r = threadIdx.x; r < nr; r += MT) {
        cplx acc = cmk(0, 0);
        for (int k = 0; k < gsz; ++k) acc = cadd(acc, ld_cg(part + (int64_t)(grp * kGrp + k) * kRowsRange + r));
        gpart[r] = acc;
      }
      if (arrive_last(S + p.o_tick_a[c] + rr * (ngrp + 1) + ngrp, ngrp, &sm.flag)) {
        for (int r = threadIdx.x; r < nr; r += MT) {
          cplx acc = cmk(0, 0);
          for (int k = 0; k < ngrp; ++k) acc = cadd(acc, ld_cg(part + (int64_t)(S4 + k) * kRowsRange + r));
          a.y4[(int64_t)c * a.r3max + r0 + r] = acc;
        }
        count_and_publish(S + p.o_cnt_a[c], nrr, S + p.o_flag_a[c], E);
      }
    }
    return;
  }
  if (q.phase == 1) {
    // ---- Y3 = G3 y4: row range rr (<= 256 rows) x column split s of the r3 columns
    if (a.phase_begin <= 0) wait_flag(S + p.o_flag_a[c], E, &sm.t_ready);
    const int64_t R = (int64_t)ch.r2 * a.n3l;
    const int nrr = p.nrb3[c], S3 = p.s3[c];
    const int rr = (int)(q.i / S3), s = (int)(q.i % S3);
    const int64_t r0 = blo(R, nrr, rr), r1 = blo(R, nrr, rr + 1);
    const int nr = (int)(r1 - r0);
    const int64_t c0 = blo(ch.r3, S3, s), c1 = blo(ch.r3, S3, s + 1);
    cplx* part = a.part + p.p_b[c] + (int64_t)rr * S3 * MT;
    tn2_dispatch(ch.G3, R, r0, nr, c0, c1, a.y4 + (int64_t)c * a.r3max, sm.u.tn.xs, part + (int64_t)s * MT);
    if (arrive_last(S + p.o_tick_b[c] + rr, S3, &sm.flag)) {
      for (int r = threadIdx.x; r < nr; r += MT) {
        cplx acc = cmk(0, 0);
        for (int k = 0; k < S3; ++k) acc = cadd(acc, ld_cg(part + (int64_t)k * MT + r));
        a.Y3[(int64_t)c * a.r2max * a.n3l + r0 + r] = acc;
      }
      publish(S + p.o_flag_b[c] + rr, E);
    }
    return;
  }
  if (q.phase == 2) {
    // ---- Y2 = G2 Y3: GEMM tile (mb, nb), M = r1 n2, N = n3l, K = r2
    const int gm = p.gm_f[c];
    const int nb = (int)(q.i / gm), mb = (int)(q.i % gm);
    const int64_t M = (int64_t)ch.r1 * a.n2, N = a.n3l;
    const int64_t n0 = (int64_t)nb * FTN, n1 = std::min<int64_t>(N, n0 + FTN);
    const cplx* Y3 = a.Y3 + (int64_t)c * a.r2max * a.n3l;
    if (a.phase_begin <= 1) {
      const int64_t R = (int64_t)ch.r2 * a.n3l;
      const int nrb = p.nrb3[c];
      const int64_t b0 = block_of(R, nrb, ch.r2 * n0), b1 = block_of(R, nrb, ch.r2 * n1 - 1);
      wait_flags(S + p.o_flag_b[c] + b0, (int)(b1 - b0 + 1), E, &sm.t_ready);
    }
    cplx* Y2 = a.Y2 + (int64_t)c * a.r1max * a.n2 * a.n3l;
    gemm_tile<FWA, FWB, false>(ch.G2, M, Y3, ch.r2, M, N, (int64_t)mb * FTM, n0, 0, ch.r2, sm.u.gemm,
                               Y2 + (int64_t)mb * FTM + M * n0, M);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned t = atomicAdd(S + p.o_cnt_c[c] + nb, 1u);
      if (t == (unsigned)gm - 1) {
        S[p.o_cnt_c[c] + nb] = 0;
        __threadfence();
        st_release(S + p.o_flag_c[c] + nb, E);
      }
    }
    return;
  }
  // ---- y = G1 Y2 over voxel columns [c0, c1) of (i2 + n2 i3)
  const int64_t ncol = (int64_t)a.n2 * a.n3l;
  const int64_t c0 = q.i * p.ecols, c1 = std::min<int64_t>(ncol, c0 + p.ecols);
  if (a.phase_begin <= 2) {
    const int64_t nb0 = (c0 / a.n2) / FTN, nb1 = ((c1 - 1) / a.n2) / FTN;
    wait_flags(S + p.o_flag_c[c] + nb0, (int)(nb1 - nb0 + 1), E, &sm.t_ready);
  }
  const cplx* Y2 = a.Y2 + (int64_t)c * a.r1max * a.n2 * a.n3l;
  cplx* y = a.y + (int64_t)c * a.chi_stride + a.vox_off;
  const int KT = (ch.r1 + 3) / 4;
  switch (KT) {
    case 1: exp_tile<1>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
    case 2: exp_tile<2>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
    case 3: exp_tile<3>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
    case 4: exp_tile<4>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
    case 5: exp_tile<5>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
    case 6: exp_tile<6>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
    case 7: exp_tile<7>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
    default: exp_tile<8>(ch.G1, a.n1, ch.r1, Y2, c0, c1, y, dyn); break;
  }
}

// ------------------------------------------------------------------ transpose tiles
__device__ __noinline__ void adj_tile(const MegaArgs& a, const Q q, unsigned E, MegaSmem& sm, cplx* dyn) {
  const MegaPlan& p = a.p;
  const int c = q.chi;
  const MegaChi& ch = a.c[c];
  unsigned* S = a.sync;
  if (q.phase == 0) {
    // ---- W1 = G1^T u over voxel columns [c0, c1)
    const int64_t ncol = (int64_t)a.n2 * a.n3l;
    const int64_t c0 = q.i * p.ecols, c1 = std::min<int64_t>(ncol, c0 + p.ecols);
    const cplx* u = a.x + (int64_t)c * a.chi_stride + a.vox_off;
    cplx* W1 = a.Y2 + (int64_t)c * a.r1max * a.n2 * a.n3l;
    const int NT = (ch.r1 + 7) / 8;
    switch (NT) {
      case 1: red_tile<1>(ch.G1, a.n1, ch.r1, u, a.conj, c0, c1, W1, dyn); break;
      case 2: red_tile<2>(ch.G1, a.n1, ch.r1, u, a.conj, c0, c1, W1, dyn); break;
      case 3: red_tile<3>(ch.G1, a.n1, ch.r1, u, a.conj, c0, c1, W1, dyn); break;
      default: red_tile<4>(ch.G1, a.n1, ch.r1, u, a.conj, c0, c1, W1, dyn); break;
    }
    publish(S + p.o_flag_e[c] + q.i, E);
    return;
  }
  if (q.phase == 1) {
    // ---- W2 = G2^T W1: GEMM tile (mb, nb) split s, M = r2, N = n3l, K = r1 n2
    const int gm = p.gm_a[c], gs = p.gs[c];
    const int nb = (int)(q.i / (gm * gs));
    const int mb = (int)((q.i / gs) % gm), s = (int)(q.i % gs);
    const int64_t K = (int64_t)ch.r1 * a.n2, M = ch.r2, N = a.n3l;
    const int64_t n0 = (int64_t)nb * ATN, n1 = std::min<int64_t>(N, n0 + ATN);
    if (a.phase_begin <= 0) {
      const int64_t ncol = (int64_t)a.n2 * a.n3l;
      const int64_t e0 = (n0 * a.n2) / p.ecols, e1 = std::min<int64_t>(ncol - 1, n1 * a.n2 - 1) / p.ecols;
      wait_flags(S + p.o_flag_e[c] + e0, (int)(e1 - e0 + 1), E, &sm.t_ready);
    }
    const cplx* W1 = a.Y2 + (int64_t)c * a.r1max * a.n2 * a.n3l;
    const int64_t chunks = (K + GKC - 1) / GKC;
    const int64_t k0 = std::min(K, blo(chunks, gs, s) * GKC), k1 = std::min(K, blo(chunks, gs, s + 1) * GKC);
    cplx* part = a.part + p.p_g[c] + ((int64_t)(nb * gm + mb) * gs) * (ATM * ATN);
    gemm_tile<AWA, AWB, true>(ch.G2, K, W1, K, M, N, (int64_t)mb * ATM, n0, k0, k1, sm.u.gemm,
                              part + (int64_t)s * ATM * ATN, ATM);
    if (arrive_last(S + p.o_tick_g[c] + nb * gm + mb, gs, &sm.flag)) {
      cplx* W2 = a.Y3 + (int64_t)c * a.r2max * a.n3l;
      const int64_t m0 = (int64_t)mb * ATM;
      for (int e = threadIdx.x; e < ATM * ATN; e += MT) {
        const int mm = e % ATM, nn = e / ATM;
        if (m0 + mm < M && n0 + nn < N) {
          cplx acc = cmk(0, 0);
          for (int ss = 0; ss < gs; ++ss) acc = cadd(acc, ld_cg(part + (int64_t)ss * ATM * ATN + e));
          W2[(m0 + mm) + M * (n0 + nn)] = acc;
        }
      }
      count_and_publish(S + p.o_cnt_c[c] + nb, gm, S + p.o_flag_c[c] + nb, E);
    }
    return;
  }
  if (q.phase == 2) {
    // ---- z3 partial = G3[rows, cols]^T W2[rows]: row range rr, 32-column chunk cc
    const int nrr = p.nrr3[c], ncc = p.ncc3[c];
    const int rr = (int)(q.i / ncc), cc = (int)(q.i % ncc);
    const int64_t R = (int64_t)ch.r2 * a.n3l;
    const int64_t r0 = blo(R, nrr, rr), r1 = blo(R, nrr, rr + 1);
    const int nrows = (int)(r1 - r0);
    const int col0 = 32 * cc, ncols = std::min(32, ch.r3 - col0);
    if (a.phase_begin <= 1) {
      const int64_t nb0 = (r0 / ch.r2) / ATN, nb1 = ((r1 - 1) / ch.r2) / ATN;
      wait_flags(S + p.o_flag_c[c] + nb0, (int)(nb1 - nb0 + 1), E, &sm.t_ready);
    }
    const cplx* W2 = a.Y3 + (int64_t)c * a.r2max * a.n3l;
    __syncthreads();
    const int npad = ((nrows + 127) / 128) * 128;
    for (int r = threadIdx.x; r < npad; r += MT) sm.u.tt.vs[r] = r < nrows ? ld_cg(W2 + r0 + r) : cmk(0, 0);
    __syncthreads();
    tt_cols(ch.G3, R, r0, nrows, col0, ncols, sm.u.tt.vs, sm.u.tt.res);
    __syncthreads();
    cplx* part = a.part + p.p_z[c] + (int64_t)cc * nrr * 32;
    if (threadIdx.x < ncols) part[(int64_t)rr * 32 + threadIdx.x] = sm.u.tt.res[threadIdx.x];
    if (arrive_last(S + p.o_tick_z[c] + cc, nrr, &sm.flag)) {
      if (threadIdx.x < ncols) {
        cplx acc = cmk(0, 0);
        for (int k = 0; k < nrr; ++k) acc = cadd(acc, ld_cg(part + (int64_t)k * 32 + threadIdx.x));
        a.y4[(int64_t)c * a.r3max + col0 + threadIdx.x] = acc;
      }
      count_and_publish(S + p.o_cnt_z[c], ncc, S + p.o_flag_z[c], E);
    }
    return;
  }
  // ---- z_chi = G4^T z3 over a column chunk, then the Eq. 18 chi sum by the last chi
  const int64_t c0 = q.i * p.cc4, c1 = std::min<int64_t>(a.mloc, c0 + p.cc4);
  if (a.phase_begin <= 2) wait_flag(S + p.o_flag_z[c], E, &sm.t_ready);
  __syncthreads();
  const int npad = ((ch.r3 + 127) / 128) * 128;
  for (int r = threadIdx.x; r < npad; r += MT)
    sm.u.tt.vs[r] = r < ch.r3 ? ld_cg(a.y4 + (int64_t)c * a.r3max + r) : cmk(0, 0);
  __syncthreads();
  cplx* zp = a.zpart + (int64_t)c * a.mloc;
  for (int64_t cb = c0; cb < c1; cb += 64) {
    const int nc = (int)std::min<int64_t>(64, c1 - cb);
    tt_cols(ch.G4, ch.r3, 0, ch.r3, cb, nc, sm.u.tt.vs, sm.u.tt.res);
    __syncthreads();
    if (threadIdx.x < nc) zp[cb + threadIdx.x] = sm.u.tt.res[threadIdx.x];
    __syncthreads();
  }
  if (arrive_last(S + p.o_tick_s + q.i, 3, &sm.flag)) {
    for (int64_t col = c0 + threadIdx.x; col < c1; col += MT) {
      cplx v = cadd(cadd(ld_cg(a.zpart + col), ld_cg(a.zpart + a.mloc + col)), ld_cg(a.zpart + 2 * a.mloc + col));
      if (a.conj) v.y = -v.y;
      a.y[col] = v;
    }
  }
}

template <bool FWD>
__global__ void __launch_bounds__(MT, MEGA_MIN_BLOCKS) k_mega(const __grid_constant__ MegaArgs a) {
  // dynamic shared memory: [MegaSmem][G1 fragments of the EXP / RED tiles]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MegaSmem& sm = *reinterpret_cast<MegaSmem*>(smem_raw);
  cplx* dyn = reinterpret_cast<cplx*>(smem_raw + ((sizeof(MegaSmem) + 127) / 128) * 128);
  __shared__ int s_tile;
  unsigned* S = a.sync;
  const unsigned E = S[2] + 1u;
  const int64_t t0 = a.p.seg_off[0], t1 = a.p.seg_off[a.p.nseg];
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(S, 1u);
    __syncthreads();
    const int64_t t = t0 + s_tile;
    __syncthreads();
    if (t >= t1) break;
    const Q q = decode(a.p, t);
    uint64_t tt0 = 0;
    if (a.trace && threadIdx.x == 0) {
      tt0 = globaltimer_ns();
      sm.t_ready = tt0;
    }
    if (FWD)
      fwd_tile(a, q, E, sm, dyn);
    else
      adj_tile(a, q, E, sm, dyn);
    if (a.trace && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.trace[4 * t] = tt0;
      a.trace[4 * t + 1] = globaltimer_ns();
      a.trace[4 * t + 2] = smid;
      a.trace[4 * t + 3] = sm.t_ready;
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned d = atomicAdd(S + 1, 1u);
    if (d == gridDim.x - 1) {
      S[0] = 0;
      S[1] = 0;
      __threadfence();
      S[2] = E;
    }
  }
}

int occupancy_grid(const void* fn, size_t dyn_smem) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, MT, dyn_smem));
  return sms * std::max(1, occ);
}

}  // namespace

// ------------------------------------------------------------------ host: plan
static size_t dyn_smem_bytes(const MegaArgs& a, bool forward) {
  size_t b = 0;
  const size_t base = ((sizeof(MegaSmem) + 127) / 128) * 128;
  for (int c = 0; c < 3; ++c) {
    const int r1 = a.c[c].r1;
    if (forward)
      b = std::max(b, (size_t)((a.n1 + 7) / 8) * ((r1 + 3) / 4) * 32 * sizeof(cplx));
    else
      b = std::max(b, (size_t)((a.n1 + 3) / 4) * ((r1 + 7) / 8) * 32 * sizeof(cplx));
  }
  return base + b;
}

void mega_plan(MegaArgs& a) {
  MegaPlan& p = a.p;
  p = MegaPlan{};
  for (int c = 0; c < 3; ++c) {
    const MegaChi& ch = a.c[c];
    VSIE_REQUIRE(ch.r3 <= 2048, VSIE_ERR_ARG, "single-RHS apply: r3 > 2048 not supported");
    VSIE_REQUIRE(ch.r1 <= 32, VSIE_ERR_ARG, "single-RHS apply: r1 > 32 not supported");
  }
  // launch geometry first (resolved here, outside any stream capture): tiles are sized
  // so that every streaming phase has >= ~2 tiles per resident CTA
  p.smem_fwd = (int)dyn_smem_bytes(a, true);
  p.smem_adj = (int)dyn_smem_bytes(a, false);
  VSIE_REQUIRE(p.smem_fwd <= 200 * 1024 && p.smem_adj <= 200 * 1024, VSIE_ERR_ARG,
               "single-RHS apply: n1 * r1 too large for shared memory");
  VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_mega<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_mega<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  p.grid_fwd = occupancy_grid((const void*)k_mega<true>, p.smem_fwd);
  p.grid_adj = occupancy_grid((const void*)k_mega<false>, p.smem_adj);
  const int64_t G = std::max(p.grid_fwd, p.grid_adj);
  static const int tpc = [] {
    const char* e = std::getenv("VSIE_MEGA_TPC");   // tiles per resident CTA per phase (tuning)
    return e ? std::max(1, std::atoi(e)) : 2;
  }();
  const int64_t per_chi = ceil_div(tpc * G, 3);   // tiles per (phase, chi) target
  int words = 3;
  int64_t elems = 0;
  auto W = [&](int n) { const int o = words; words += n; return o; };
  const int64_t ncol = (int64_t)a.n2 * a.n3l;
  p.ecols = (int)std::max<int64_t>(64, ceil_div(ceil_div(ncol, per_chi), 64) * 64);
  p.ne = (int)ceil_div(ncol, p.ecols);
  p.gn_f = (int)ceil_div(a.n3l, FTN);
  p.gn_a = (int)ceil_div(a.n3l, ATN);
  p.cc4 = (int)std::max<int64_t>(16, ceil_div(ceil_div(a.mloc, per_chi), 16) * 16);
  p.ncc4 = (int)ceil_div(a.mloc, p.cc4);
  for (int c = 0; c < 3; ++c) {
    const MegaChi& ch = a.c[c];
    const int64_t R3 = (int64_t)ch.r2 * a.n3l;
    // forward phase 0: row ranges (<= 1024 rows, whole columns when r3 <= 1024) x column
    // splits (~per_chi tiles; a tile's x range fits the smem stage)
    p.nrb4[c] = (int)ceil_div(ch.r3, kRowsRange);
    p.s4[c] = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(per_chi, p.nrb4[c]), std::max<int64_t>(1, a.mloc / 16)));
    p.s4[c] = (int)std::max<int64_t>(p.s4[c], ceil_div(a.mloc, 2048));
    // forward phase 1: row ranges of <= 256 rows x column splits of the r3 columns
    p.nrb3[c] = (int)std::max<int64_t>(1, ceil_div(R3, MT));
    p.s3[c] = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(per_chi, p.nrb3[c]), ceil_div(ch.r3, 16)));
    // GEMM tiles: forward M = r1 n2 (64 x 32); transpose M = r2 (32 x 64, split-K over r1 n2)
    p.gm_f[c] = (int)ceil_div((int64_t)ch.r1 * a.n2, FTM);
    p.gm_a[c] = (int)ceil_div(ch.r2, ATM);
    const int64_t chunks = ceil_div((int64_t)ch.r1 * a.n2, GKC);
    p.gs[c] = (int)std::max<int64_t>(1, std::min<int64_t>(chunks / 4, ceil_div(per_chi, (int64_t)p.gm_a[c] * p.gn_a)));
    // transpose phase 2: row ranges (<= 1024 rows) x 32-column chunks
    p.ncc3[c] = (int)ceil_div(ch.r3, 32);
    p.nrr3[c] = (int)std::max<int64_t>(1, std::max(ceil_div(R3, kRowsTT), std::min(ceil_div(R3, 128), ceil_div(per_chi, p.ncc3[c]))));
    // sync words
    p.o_tick_a[c] = W(p.nrb4[c] * ((p.s4[c] + kGrp - 1) / kGrp + 1));
    p.o_tick_b[c] = W(p.nrb3[c]);
    p.o_cnt_a[c] = W(1);
    p.o_flag_a[c] = W(1);
    p.o_flag_b[c] = W(p.nrb3[c]);
    p.o_cnt_c[c] = W(std::max(p.gn_f, p.gn_a));
    p.o_flag_c[c] = W(std::max(p.gn_f, p.gn_a));
    p.o_flag_e[c] = W(p.ne);
    p.o_tick_g[c] = W(p.gn_a * p.gm_a[c]);
    p.o_tick_z[c] = W(p.ncc3[c]);
    p.o_cnt_z[c] = W(1);
    p.o_flag_z[c] = W(1);
    // partials
    p.p_a[c] = elems;
    elems += (int64_t)p.nrb4[c] * (p.s4[c] + (p.s4[c] + kGrp - 1) / kGrp) * kRowsRange;
    p.p_b[c] = elems;
    elems += (int64_t)p.nrb3[c] * p.s3[c] * MT;
    p.p_g[c] = elems;
    elems += (int64_t)p.gn_a * p.gm_a[c] * p.gs[c] * ATM * ATN;
    p.p_z[c] = elems;
    elems += (int64_t)p.ncc3[c] * p.nrr3[c] * 32;
  }
  p.o_tick_s = W(p.ncc4);
  p.sync_words = words;
  p.part_elems = elems;
}

std::vector<MegaTraceRec> mega_decode_trace(const MegaPlan& p, const unsigned long long* tr) {
  std::vector<MegaTraceRec> out;
  const int64_t n = p.seg_off[p.nseg];
  unsigned long long tmin = ~0ull;
  for (int64_t t = 0; t < n; ++t)
    if (tr[4 * t]) tmin = std::min(tmin, tr[4 * t]);
  for (int s = 0; s < p.nseg; ++s)
    for (int64_t t = p.seg_off[s]; t < p.seg_off[s + 1]; ++t) {
      MegaTraceRec r;
      r.phase = p.seg_phase[s];
      r.chi = p.seg_chi[s];
      r.idx = t - p.seg_off[s];
      r.sm = (int)tr[4 * t + 2];
      r.t0_us = (double)(tr[4 * t] - tmin) * 1e-3;
      r.t1_us = (double)(tr[4 * t + 1] - tmin) * 1e-3;
      r.tr_us = (double)(tr[4 * t + 3] - tmin) * 1e-3;
      out.push_back(r);
    }
  return out;
}

void launch_mega(const MegaArgs& args, bool forward, cudaStream_t st, MegaPlan* plan_out) {
  MegaArgs a = args;
  MegaPlan& p = a.p;
  for (int c = 0; c < 3; ++c) {
    p.count[0][c] = forward ? p.nrb4[c] * p.s4[c] : p.ne;
    p.count[1][c] = forward ? p.nrb3[c] * p.s3[c] : p.gn_a * p.gm_a[c] * p.gs[c];
    p.count[2][c] = forward ? p.gn_f * p.gm_f[c] : p.nrr3[c] * p.ncc3[c];
    p.count[3][c] = forward ? p.ne : p.ncc4;
  }
  // claim order: diagonal over (phase, chi) so that HBM-bound steps of one chi run
  // beside the tensor-core steps of another; (phase, chi) always after (phase-1, chi)
  p.nseg = 0;
  int off = 0;
  static const int diag = [] {
    const char* e = std::getenv("VSIE_MEGA_ORDER");
    return e ? std::atoi(e) : 0;
  }();
  for (int d = 0; d < kMegaPhases + 2; ++d)
    for (int c = 0; c < 3; ++c) {
      const int ph = diag ? d - c : d;
      if (!diag && d >= kMegaPhases) continue;
      if (ph < 0 || ph >= kMegaPhases || ph < a.phase_begin || ph >= a.phase_end) continue;
      p.seg_phase[p.nseg] = ph;
      p.seg_chi[p.nseg] = c;
      p.seg_off[p.nseg] = off;
      off += p.count[ph][c];
      ++p.nseg;
    }
  p.seg_off[p.nseg] = off;
  if (p.nseg == 0 || off == 0) return;
  if (plan_out) *plan_out = p;
  if (forward)
    k_mega<true><<<std::min(p.grid_fwd, off), MT, p.smem_fwd, st>>>(a);
  else
    k_mega<false><<<std::min(p.grid_adj, off), MT, p.smem_adj, st>>>(a);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
