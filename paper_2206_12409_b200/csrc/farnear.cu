// The far-near conductor block Z_cc^fn of the hybrid VSIE: its entries
// (Eq. 11: Galerkin interactions between the near and the far RWG functions), its
// ACA compression U V^* = ACA(Z_cc^fn) (Eq. 12) and the two low-rank products of
// every GMRES matvec, U V^* j_f and V-bar U^T j_n (Eq. 15).  W = conj(V) is stored,
// so Z^fn ~= U W^T and (Z^fn)^T ~= W U^T.  Contract: include/vsie_farnear.h.
//
// Kernels:
//  * cc_entry: 36 pair interactions J_p . (G(r_p - r_s) J_s) per entry, FP64, one rsqrt and one
//    sincos per pair (the near and far surfaces are separated, so no Taylor phase: the triangle
//    quadrature nodes span k0 |d| ~ 0.1 rad, too wide for a short series at 1e-16).
//  * k_aca: the whole partially pivoted ACA as ONE cooperative persistent kernel.  A step is
//    sequential (each row / column depends on every earlier term), and a host-driven loop would
//    pay ~6 launches and a device->host pivot read per step; here a step is three grid-wide
//    barriers: (A) residual row on the entry kernel + column argmax partials, (B) w_k, residual
//    column u_k, ||u||, ||w|| and the next-row argmax partials, (C) the cross terms
//    (U_l^H u_k)(W_l^H w_k) of the Frobenius-norm recursion, chunked over blocks; every block
//    then reduces the partials itself in a fixed order (no atomics: bitwise reproducible).
//    Buffers written inside the kernel are read with ld.global.cg (L2, never a stale L1 line).
//  * k_lr_dot / k_lr_expand: the low-rank apply y = F2 (F1^T x) as two HBM-streaming launches
//    (one per factor) chained with PDL; the pair of Eq. 15 runs both products in the same two
//    launches.  Split-K partials of the dots are summed by the last CTA of each l-group in a
//    fixed order.  nrhs > 1 runs on the DMMA ZGEMM (linalg.cu).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>

#include "crosskern.cuh"
#include "farnear.hpp"
#include "geometry.hpp"

namespace cg = cooperative_groups;

namespace vsie {

namespace {

constexpr double kInv4Pi = 0.079577471545947667884;   // 1 / (4 pi)

struct CcGeom {
  const double* a;   // near [ma][36]
  const double* b;   // far  [mb][36]
  int64_t ma, mb;
  double k0, inv_k0, scale_re, scale_im;
};

// Z^fn[i, j]: sum over the 6 x 6 node pairs of J_p . G(R) J_s with
//   J_p . G J_s = g [alpha (J_p . J_s) + beta (J_p . Rhat)(Rhat . J_s)],
//   alpha = 1 - i u - u^2, beta = -1 + 3 i u + 3 u^2, u = 1 / (k0 R), g = exp(-i k0 R) / (4 pi R).
__device__ __forceinline__ cplx cc_entry(const CcGeom& g, int64_t i, int64_t j) {
  const double* A = g.a + 36 * i;
  const double* B = g.b + 36 * j;
  double ar = 0, ai = 0;
#pragma unroll 1
  for (int p = 0; p < 6; ++p) {
    const double px = __ldg(A + 6 * p), py = __ldg(A + 6 * p + 1), pz = __ldg(A + 6 * p + 2);
    const double jpx = __ldg(A + 6 * p + 3), jpy = __ldg(A + 6 * p + 4), jpz = __ldg(A + 6 * p + 5);
#pragma unroll 2
    for (int s = 0; s < 6; ++s) {
      const double rx = px - __ldg(B + 6 * s), ry = py - __ldg(B + 6 * s + 1), rz = pz - __ldg(B + 6 * s + 2);
      const double jsx = __ldg(B + 6 * s + 3), jsy = __ldg(B + 6 * s + 4), jsz = __ldg(B + 6 * s + 5);
      const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
      const double ir = rsqrt(r2);
      double sn, cs;
      sincos(g.k0 * (r2 * ir), &sn, &cs);
      const double u = g.inv_k0 * ir, u2 = u * u;
      const double jj = fma(jpx, jsx, fma(jpy, jsy, jpz * jsz));
      const double t = fma(jpx, rx, fma(jpy, ry, jpz * rz)) * fma(rx, jsx, fma(ry, jsy, rz * jsz)) * (ir * ir);
      const double re = fma(1.0 - u2, jj, (3.0 * u2 - 1.0) * t);
      const double im = u * (3.0 * t - jj);
      // (cs - i sn)(re + i im) / R
      ar = fma(ir, fma(cs, re, sn * im), ar);
      ai = fma(ir, fma(cs, im, -sn * re), ai);
    }
  }
  ar *= kInv4Pi;
  ai *= kInv4Pi;
  return cmk(g.scale_re * ar - g.scale_im * ai, g.scale_re * ai + g.scale_im * ar);
}

__device__ __forceinline__ cplx ldcg(const cplx* p) { return __ldcg(p); }

__global__ void __launch_bounds__(256) k_cc_list(CcGeom g, const int64_t* __restrict__ idx, int64_t count,
                                                 cplx* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = cc_entry(g, idx[2 * t], idx[2 * t + 1]);
}

// min over near x far quadrature nodes of |r_p - r_s|, as the bits of a positive double
// (monotone as unsigned 64-bit integers) through atomicMin
__global__ void __launch_bounds__(256) k_min_dist(const double* __restrict__ a, int64_t na, const double* __restrict__ b,
                                                  int64_t nb, unsigned long long* out) {
  __shared__ double sb[3 * 256];
  double best = 1e300;
  const int64_t ia = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // near node id (RWG * 6 + q)
  double x = 0, y = 0, z = 0;
  if (ia < na) {
    x = a[6 * ia];
    y = a[6 * ia + 1];
    z = a[6 * ia + 2];
  }
  for (int64_t j0 = (int64_t)blockIdx.y * 256; j0 < nb; j0 += (int64_t)gridDim.y * 256) {
    __syncthreads();
    const int64_t jb = j0 + threadIdx.x;
    if (jb < nb) {
      sb[3 * threadIdx.x] = b[6 * jb];
      sb[3 * threadIdx.x + 1] = b[6 * jb + 1];
      sb[3 * threadIdx.x + 2] = b[6 * jb + 2];
    }
    __syncthreads();
    const int lim = (int)std::min<int64_t>(256, nb - j0);
    if (ia < na)
      for (int q = 0; q < lim; ++q) {
        const double dx = x - sb[3 * q], dy = y - sb[3 * q + 1], dz = z - sb[3 * q + 2];
        best = fmin(best, fma(dx, dx, fma(dy, dy, dz * dz)));
      }
  }
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && ia - (threadIdx.x & 31) < na)
    atomicMin(out, (unsigned long long)__double_as_longlong(sqrt(best)));
}

// ------------------------------------------------------------------ ACA (one cooperative kernel)
constexpr int kAcaThreads = 256;

struct AcaOut {
  int k, stop;
  double norm2, last2;
  long long entries;
};

struct AcaArgs {
  CcGeom g;
  cplx* U;                 // [kmax][m] (column l at U + l m)
  cplx* W;                 // [kmax][n]
  int64_t m, n;
  int kmax;
  double tol2;
  cplx* rrow;              // [n]
  unsigned char* used;     // [m]
  double* bval;            // [G] phase A: per-block max |rrow|^2
  long long* bidx;
  double* bu2;             // [G] phase B: ||u||^2, ||w||^2, max |u|^2 over unused rows
  double* bw2;
  double* bumax;
  long long* buidx;
  cplx* pc;                // [kmax][G] phase C: chunk partials of U_l^H u_k
  cplx* pd;                // [kmax][G] and of W_l^H w_k
  int* piv_i;
  int* piv_j;
  AcaOut* out;
};

// (value, index) argmax over the block: larger value wins, ties -> smaller index
__device__ void block_argmax(double& v, long long& i, double* sv, long long* si) {
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
    sv[w] = v;
    si[w] = i;
  }
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sv[lane] : -2.0;
    i = lane < (int)(blockDim.x >> 5) ? si[lane] : LLONG_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
      if (v2 > v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
      }
    }
    if (lane == 0) {
      sv[0] = v;
      si[0] = i;
    }
  }
  __syncthreads();
  v = sv[0];
  i = si[0];
}

// sum of NV doubles per thread over the block (fixed tree), result in every thread
template <int NV>
__device__ void block_sum(double (&v)[NV], double* sv) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) sv[q * 32 + w] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0;
    for (int x = 0; x < nw; ++x) s += sv[q * 32 + x];
    v[q] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void csub_mul(cplx& v, cplx a, cplx b) {   // v -= a b
  v.x = fma(-a.x, b.x, v.x);
  v.x = fma(a.y, b.y, v.x);
  v.y = fma(-a.x, b.y, v.y);
  v.y = fma(-a.y, b.x, v.y);
}

__device__ __forceinline__ void cfma_conj(cplx& acc, cplx a, cplx b) {   // acc += conj(a) b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

__global__ void __launch_bounds__(kAcaThreads) k_aca(AcaArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[4 * 32];
  __shared__ long long si[32];
  const int G = gridDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)G * blockDim.x;
  const int64_t m = a.m, n = a.n;
  int k = 0, stop = -1;
  int64_t i = 0;
  double norm2 = 0, last2 = 0;
  long long entries = 0;
  for (;;) {
    if (k >= a.kmax) {
      stop = 1;
      break;
    }
    // (A) residual row r = Z[i, :] - sum_l U[i, l] w_l and its argmax partials
    double best = -1.0;
    long long bj = LLONG_MAX;
    for (int64_t j = tid; j < n; j += nth) {
      cplx v = cc_entry(a.g, i, j);
#pragma unroll 4
      for (int l = 0; l < k; ++l) csub_mul(v, ldcg(a.U + l * m + i), ldcg(a.W + l * n + j));
      a.rrow[j] = v;
      const double mag = cabs2(v);
      if (mag > best) {
        best = mag;
        bj = j;
      }
    }
    block_argmax(best, bj, sv, si);
    if (threadIdx.x == 0) {
      a.bval[blockIdx.x] = best;
      a.bidx[blockIdx.x] = bj;
    }
    if (tid == 0) a.used[i] = 1;
    entries += n;
    grid.sync();
    // (B) column pivot j_k (every block reduces the G partials in the same order)
    best = -1.0;
    bj = LLONG_MAX;
    for (int b = threadIdx.x; b < G; b += blockDim.x) {
      const double v = __ldcg(a.bval + b);
      const long long jj = __ldcg(a.bidx + b);
      if (v > best || (v == best && jj < bj)) {
        best = v;
        bj = jj;
      }
    }
    block_argmax(best, bj, sv, si);
    if (!(best > 0.0)) {
      // the residual row vanishes: take the smallest unused row (the used row stays used)
      double v = -1.0;
      long long r = LLONG_MAX;
      for (int64_t q = threadIdx.x; q < m; q += blockDim.x)
        if (!__ldcg(a.used + q)) {
          v = 0.0;
          r = q;
          break;
        }
      block_argmax(v, r, sv, si);
      if (v < 0) {
        stop = 2;
        break;
      }
      i = r;
      grid.sync();   // nobody rewrites rrow / the partials while a peer still reads them
      continue;
    }
    const int64_t jk = bj;
    const cplx piv = ldcg(a.rrow + jk);
    const double ip = 1.0 / cabs2(piv);
    const cplx inv = cmk(piv.x * ip, -piv.y * ip);
    double acc[2] = {0, 0};   // ||w||^2, ||u||^2
    for (int64_t j = tid; j < n; j += nth) {
      const cplx w = cmul(ldcg(a.rrow + j), inv);
      a.W[k * n + j] = w;
      acc[0] += cabs2(w);
    }
    double umax = -1.0;
    long long ui = LLONG_MAX;
    for (int64_t r = tid; r < m; r += nth) {
      cplx v = cc_entry(a.g, r, jk);
#pragma unroll 4
      for (int l = 0; l < k; ++l) csub_mul(v, ldcg(a.U + l * m + r), ldcg(a.W + l * n + jk));
      a.U[k * m + r] = v;
      const double mag = cabs2(v);
      acc[1] += mag;
      if (!__ldcg(a.used + r) && mag > umax) {
        umax = mag;
        ui = r;
      }
    }
    entries += m;
    block_sum<2>(acc, sv);
    block_argmax(umax, ui, sv, si);
    if (threadIdx.x == 0) {
      a.bw2[blockIdx.x] = acc[0];
      a.bu2[blockIdx.x] = acc[1];
      a.bumax[blockIdx.x] = umax;
      a.buidx[blockIdx.x] = ui;
    }
    if (tid == 0) {
      a.piv_i[k] = (int)i;
      a.piv_j[k] = (int)jk;
    }
    grid.sync();
    // (C) chunk partials of U_l^H u_k and W_l^H w_k, l < k: C chunks per l
    const int C = k > 0 ? std::max(1, G / k) : 1;
    for (int item = blockIdx.x; item < k * C; item += G) {
      const int l = item / C, c = item % C;
      double cd[4] = {0, 0, 0, 0};
      cplx s = cmk(0, 0), d = cmk(0, 0);
      for (int64_t r = m * c / C + threadIdx.x; r < m * (c + 1) / C; r += blockDim.x)
        cfma_conj(s, ldcg(a.U + l * m + r), ldcg(a.U + k * m + r));
      for (int64_t j = n * c / C + threadIdx.x; j < n * (c + 1) / C; j += blockDim.x)
        cfma_conj(d, ldcg(a.W + l * n + j), ldcg(a.W + k * n + j));
      cd[0] = s.x;
      cd[1] = s.y;
      cd[2] = d.x;
      cd[3] = d.y;
      block_sum<4>(cd, sv);
      if (threadIdx.x == 0) {
        a.pc[(int64_t)l * G + c] = cmk(cd[0], cd[1]);
        a.pd[(int64_t)l * G + c] = cmk(cd[2], cd[3]);
      }
    }
    grid.sync();
    // (D) norm recursion, stop test and the next row (every block, same order)
    double nrm[3] = {0, 0, 0};   // ||u||^2, ||w||^2, sum_l Re(c_l d_l)
    for (int b = threadIdx.x; b < G; b += blockDim.x) {
      nrm[0] += __ldcg(a.bu2 + b);
      nrm[1] += __ldcg(a.bw2 + b);
    }
    for (int l = threadIdx.x; l < k; l += blockDim.x) {
      cplx s = cmk(0, 0), d = cmk(0, 0);
      for (int c = 0; c < C; ++c) {
        s = cadd(s, ldcg(a.pc + (int64_t)l * G + c));
        d = cadd(d, ldcg(a.pd + (int64_t)l * G + c));
      }
      nrm[2] += s.x * d.x - s.y * d.y;
    }
    block_sum<3>(nrm, sv);
    last2 = nrm[0] * nrm[1];
    norm2 += 2.0 * nrm[2] + last2;
    ++k;
    if (last2 <= a.tol2 * norm2) {
      stop = 0;
      break;
    }
    umax = -1.0;
    ui = LLONG_MAX;
    for (int b = threadIdx.x; b < G; b += blockDim.x) {
      const double v = __ldcg(a.bumax + b);
      const long long r = __ldcg(a.buidx + b);
      if (v > umax || (v == umax && r < ui)) {
        umax = v;
        ui = r;
      }
    }
    block_argmax(umax, ui, sv, si);
    if (umax < 0) {
      stop = 2;
      break;
    }
    i = ui;
  }
  if (tid == 0) {
    a.out->k = k;
    a.out->stop = stop;
    a.out->norm2 = norm2;
    a.out->last2 = last2;
    a.out->entries = entries;
  }
}

// ------------------------------------------------------------------ low-rank apply (nrhs = 1)
constexpr int kRCMax = 4096;  // max rows per chunk of a dot block (x chunk staged in smem)
constexpr int kLB = 32;       // l per dot block (4 per warp)
constexpr int kExpRows = 32;  // rows per expand block (one per lane; the 8 warps split l)

struct LrJob {
  const cplx* F;    // [k][dim]
  int64_t dim;
  const cplx* x;    // dot input [dim]
  cplx* y;          // expand output [dim]
  int conj;
  int rc;           // dot: rows per chunk
  int nchunk;       // dot: chunks
};

struct LrArgs {
  LrJob dot[2];     // t[j] = op(dot[j].F)^T dot[j].x
  LrJob exp[2];     // exp[j].y = op(exp[j].F) t[j]
  int njob, k, lgroups;
  int64_t cmax;     // max nchunk (part stride)
  cplx* part;       // [job][l][chunk]
  cplx* t;          // [job][k]
  unsigned* counters;   // [job][lgroups]
};

__device__ __forceinline__ cplx opF(cplx v, int conj) { return conj ? cconj(v) : v; }

// t[job][l] = sum_r op(F[l dim + r]) x[r]: block = (chunk of rc rows, 32 l); warp w takes
// l = 32 lg + w + 8 q (q < 4), lanes stride the rows (coalesced 512-B column segments);
// the last block of each (job, l-group) sums the chunk partials in chunk order
__global__ void __launch_bounds__(256) k_lr_dot(LrArgs a) {
  extern __shared__ cplx xs[];
  __shared__ bool last;
  __shared__ cplx sl[8][32];
  int b = blockIdx.x;
  const int per0 = a.dot[0].nchunk * a.lgroups;
  const int job = b < per0 ? 0 : 1;
  if (job == 1) b -= per0;
  const LrJob& J = a.dot[job];
  const int chunk = b % J.nchunk, lg = b / J.nchunk;
  const int64_t r0 = (int64_t)chunk * J.rc, r1 = std::min<int64_t>(J.dim, r0 + J.rc);
  pdl_wait();
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) xs[r - r0] = J.x[r];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lbase = lg * kLB + w;
  cplx acc[4];
  const cplx* Fl[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    acc[q] = cmk(0, 0);
    const int l = std::min(lbase + 8 * q, a.k - 1);
    Fl[q] = J.F + (int64_t)l * J.dim;
  }
#pragma unroll 2
  for (int64_t r = r0 + lane; r < r1; r += 32) {
    const cplx xv = xs[r - r0];
#pragma unroll
    for (int q = 0; q < 4; ++q) cfma(acc[q], opF(__ldg(Fl[q] + r), J.conj), xv);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    for (int o = 16; o > 0; o >>= 1) {
      acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
      acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
    }
    const int l = lbase + 8 * q;
    if (lane == 0 && l < a.k) a.part[((int64_t)job * a.k + l) * a.cmax + chunk] = acc[q];
  }
  pdl_trigger();
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ctr = a.counters + job * a.lgroups + lg;
    last = atomicAdd(ctr, 1u) == (unsigned)J.nchunk - 1;
    if (last) *ctr = 0;   // ready for the next launch (graph replays)
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // 256 threads: l = 32 lg + (tid % 32), slice s = tid / 32 sums chunks s, s + 8, ...
  const int li = threadIdx.x & 31, s = threadIdx.x >> 5;
  const int l = lg * kLB + li;
  cplx v = cmk(0, 0);
  if (l < a.k)
    for (int c = s; c < J.nchunk; c += 8) v = cadd(v, __ldcg(a.part + ((int64_t)job * a.k + l) * a.cmax + c));
  sl[s][li] = v;
  __syncthreads();
  if (s == 0 && l < a.k) {
    cplx tot = sl[0][li];
    for (int q = 1; q < 8; ++q) tot = cadd(tot, sl[q][li]);
    a.t[(int64_t)job * a.k + l] = tot;
  }
}

// y[r] = sum_l op(F[l dim + r]) t[l]: block = 32 rows (one per lane), warp w takes l = w + 8 q,
// the 8 warp partials are summed in warp order
__global__ void __launch_bounds__(256) k_lr_expand(LrArgs a) {
  extern __shared__ cplx ts[];
  __shared__ cplx red[8][kExpRows];
  int b = blockIdx.x;
  const int per0 = (int)ceil_div(a.exp[0].dim, kExpRows);
  const int job = b < per0 ? 0 : 1;
  if (job == 1) b -= per0;
  const LrJob& J = a.exp[job];
  pdl_wait();
  for (int l = threadIdx.x; l < a.k; l += blockDim.x) ts[l] = __ldcg(a.t + (int64_t)job * a.k + l);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)b * kExpRows + lane;
  cplx acc0 = cmk(0, 0), acc1 = cmk(0, 0);
  if (r < J.dim) {
    const cplx* F = J.F + r;
    int l = w;
#pragma unroll 4
    for (; l + 8 < a.k; l += 16) {
      cfma(acc0, opF(__ldg(F + (int64_t)l * J.dim), J.conj), ts[l]);
      cfma(acc1, opF(__ldg(F + (int64_t)(l + 8) * J.dim), J.conj), ts[l + 8]);
    }
    if (l < a.k) cfma(acc0, opF(__ldg(F + (int64_t)l * J.dim), J.conj), ts[l]);
  }
  red[w][lane] = cadd(acc0, acc1);
  pdl_trigger();
  __syncthreads();
  if (w == 0 && r < J.dim) {
    cplx tot = red[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) tot = cadd(tot, red[q][lane]);
    J.y[r] = tot;
  }
}

int aca_grid(const void* kernel) {
  int dev = 0, nsm = 0, per = 0;
  VSIE_CHECK_CUDA(cudaGetDevice(&dev));
  VSIE_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kAcaThreads, 0));
  VSIE_REQUIRE(per >= 1, VSIE_ERR_CUDA, "k_aca cannot be resident");
  return nsm * std::min(per, 4);
}

CcGeom geom_of(const vsie_farnear_s* h) {
  CcGeom g;
  g.a = h->src_n.p;
  g.b = h->src_f.p;
  g.ma = h->mn;
  g.mb = h->mf;
  g.k0 = h->k0;
  g.inv_k0 = 1.0 / h->k0;
  g.scale_re = h->scale_re;
  g.scale_im = h->scale_im;
  return g;
}

}  // namespace

// --------------------------------------------------------------------------- host side
int farnear_build(const vsie_mesh* near_m, int n_near, const vsie_mesh* far_m, int n_far, double freq, double tol,
                  const vsie_farnear_opts& o, vsie_farnear_s* h) {
  const auto t0 = std::chrono::steady_clock::now();
  VSIE_REQUIRE(freq > 0 && std::isfinite(freq), VSIE_ERR_ARG, "freq must be > 0");
  VSIE_REQUIRE(tol > 0 && std::isfinite(tol), VSIE_ERR_ARG, "tol must be > 0");
  VSIE_REQUIRE(o.max_rank >= 1 && o.max_rank <= 8192, VSIE_ERR_ARG, "max_rank must be in [1, 8192]");
  VSIE_REQUIRE(std::isfinite(o.scale_re) && std::isfinite(o.scale_im), VSIE_ERR_ARG, "bad scale");
  // host validation first (no CUDA call before the meshes are accepted)
  const Sources sn = build_rwg_sources(near_m, n_near);
  const Sources sf = build_rwg_sources(far_m, n_far);
  if (o.device >= 0) VSIE_CHECK_CUDA(cudaSetDevice(o.device));
  VSIE_CHECK_CUDA(cudaGetDevice(&h->device));
  h->mn = sn.m;
  h->mf = sf.m;
  VSIE_REQUIRE(h->mn < INT_MAX && h->mf < INT_MAX, VSIE_ERR_ARG, "too many RWG functions");
  h->max_edge = std::max(max_edge_length(near_m, n_near), max_edge_length(far_m, n_far));
  h->k0 = 2.0 * 3.14159265358979323846 * freq / 299792458.0;
  h->scale_re = o.scale_re;
  h->scale_im = o.scale_im;
  h->src_n.alloc(sn.table.size());
  h->src_f.alloc(sf.table.size());
  VSIE_CHECK_CUDA(cudaMemcpy(h->src_n.p, sn.table.data(), sn.table.size() * sizeof(double), cudaMemcpyHostToDevice));
  VSIE_CHECK_CUDA(cudaMemcpy(h->src_f.p, sf.table.data(), sf.table.size() * sizeof(double), cudaMemcpyHostToDevice));
  cudaStream_t st = nullptr;
  // non-singular rule (reading R-CC3): every near node at least one max-edge from every far node
  {
    DevBuf<unsigned long long> md(1);
    const double big = 1e300;
    unsigned long long init;
    std::memcpy(&init, &big, sizeof(init));
    VSIE_CHECK_CUDA(cudaMemcpy(md.p, &init, sizeof(init), cudaMemcpyHostToDevice));
    const int64_t na = 6 * h->mn, nb = 6 * h->mf;
    dim3 grid((unsigned)ceil_div(na, 256), (unsigned)std::min<int64_t>(ceil_div(nb, 256), 64));
    k_min_dist<<<grid, 256, 0, st>>>(h->src_n.p, na, h->src_f.p, nb, md.p);
    VSIE_CHECK_LAUNCH();
    unsigned long long bits;
    VSIE_CHECK_CUDA(cudaMemcpy(&bits, md.p, sizeof(bits), cudaMemcpyDeviceToHost));
    std::memcpy(&h->min_dist, &bits, sizeof(bits));
    VSIE_REQUIRE(h->min_dist >= h->max_edge, VSIE_ERR_GEOMETRY,
                 "near and far quadrature nodes closer than the longest edge (non-singular rule)");
  }
  const int kmax = (int)std::min<int64_t>(o.max_rank, std::min(h->mn, h->mf));
  const int G = aca_grid((const void*)k_aca);
  DevBuf<cplx> U((size_t)kmax * h->mn), W((size_t)kmax * h->mf), rrow(h->mf), pc((size_t)kmax * G), pd((size_t)kmax * G);
  DevBuf<unsigned char> used(h->mn);
  DevBuf<double> bval(G), bu2(G), bw2(G), bumax(G);
  DevBuf<long long> bidx(G), buidx(G);
  DevBuf<int> piv_i(kmax), piv_j(kmax);
  DevBuf<AcaOut> out(1);
  VSIE_CHECK_CUDA(cudaMemset(used.p, 0, h->mn));
  AcaArgs a;
  a.g = geom_of(h);
  a.U = U.p;
  a.W = W.p;
  a.m = h->mn;
  a.n = h->mf;
  a.kmax = kmax;
  a.tol2 = tol * tol;
  a.rrow = rrow.p;
  a.used = used.p;
  a.bval = bval.p;
  a.bidx = bidx.p;
  a.bu2 = bu2.p;
  a.bw2 = bw2.p;
  a.bumax = bumax.p;
  a.buidx = buidx.p;
  a.pc = pc.p;
  a.pd = pd.p;
  a.piv_i = piv_i.p;
  a.piv_j = piv_j.p;
  a.out = out.p;
  void* params[] = {&a};
  VSIE_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)k_aca, dim3(G), dim3(kAcaThreads), params, 0, st));
  VSIE_CHECK_LAUNCH();
  AcaOut r;
  VSIE_CHECK_CUDA(cudaMemcpy(&r, out.p, sizeof(r), cudaMemcpyDeviceToHost));
  h->rank = r.k;
  h->stop = r.stop;
  h->frob = std::sqrt(std::max(r.norm2, 0.0));
  h->est_err = r.norm2 > 0 ? std::sqrt(r.last2 / r.norm2) : 0.0;
  h->entries = r.entries;
  h->piv_i.assign(h->rank, 0);
  h->piv_j.assign(h->rank, 0);
  if (h->rank > 0) {
    VSIE_CHECK_CUDA(cudaMemcpy(h->piv_i.data(), piv_i.p, h->rank * sizeof(int), cudaMemcpyDeviceToHost));
    VSIE_CHECK_CUDA(cudaMemcpy(h->piv_j.data(), piv_j.p, h->rank * sizeof(int), cudaMemcpyDeviceToHost));
    // keep exactly rank columns (the column-major prefix of the kmax buffers)
    h->U.alloc((size_t)h->rank * h->mn);
    h->W.alloc((size_t)h->rank * h->mf);
    VSIE_CHECK_CUDA(cudaMemcpy(h->U.p, U.p, h->U.bytes(), cudaMemcpyDeviceToDevice));
    VSIE_CHECK_CUDA(cudaMemcpy(h->W.p, W.p, h->W.bytes(), cudaMemcpyDeviceToDevice));
  }
  // apply workspaces (nrhs = 1 path)
  const int k = std::max(h->rank, 1);
  const int lgroups = (int)ceil_div(k, kLB);
  const int64_t cmax = ceil_div(std::max(h->mn, h->mf), 256);
  h->part.alloc((size_t)2 * k * cmax);
  h->t.alloc((size_t)2 * k);
  h->counters.alloc((size_t)2 * lgroups);
  VSIE_CHECK_CUDA(cudaMemset(h->counters.p, 0, h->counters.bytes()));
  VSIE_CHECK_CUDA(cudaDeviceSynchronize());
  h->build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (o.verbose)
    std::fprintf(stderr, "[farnear] m_n %lld m_f %lld rank %d stop %d est_err %.3e build %.3f s\n", (long long)h->mn,
                 (long long)h->mf, h->rank, h->stop, h->est_err, h->build_s);
  return h->stop == 1 ? VSIE_WARN_NOT_CONVERGED : VSIE_OK;
}

void farnear_entries(vsie_farnear_s* h, const int64_t* idx, int64_t count, void* out, cudaStream_t st) {
  VSIE_REQUIRE(count >= 0 && (count == 0 || (idx && out)), VSIE_ERR_ARG, "entries: bad arguments");
  if (count == 0) return;
  const int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 32);
  k_cc_list<<<blocks, 256, 0, st>>>(geom_of(h), idx, count, static_cast<cplx*>(out));
  VSIE_CHECK_LAUNCH();
}

namespace {

// rows per dot chunk: about 4 CTAs per SM over the launch, in proportion to each job's rows
int dot_rows_per_chunk(int64_t dim, int64_t dim_total, int lgroups) {
  const int64_t target = std::max<int64_t>(1, (4 * 148 * dim) / (dim_total * lgroups));   // chunks wanted
  int64_t rc = ceil_div(ceil_div(dim, target), 256) * 256;
  return (int)std::min<int64_t>(kRCMax, std::max<int64_t>(256, rc));
}

// y_j = op(E_j) (op(D_j)^T x_j) for the jobs j (nrhs = 1): two launches
void lr_launch(vsie_farnear_s* h, int njob, const LrJob* dot, const LrJob* exp, cudaStream_t st) {
  LrArgs a{};
  a.njob = njob;
  a.k = h->rank;
  a.lgroups = (int)ceil_div(h->rank, kLB);
  a.part = h->part.p;
  a.t = h->t.p;
  a.counters = h->counters.p;
  int64_t dim_total = 0;
  for (int j = 0; j < njob; ++j) dim_total += dot[j].dim;
  int dot_blocks = 0, exp_blocks = 0, rc_max = 0;
  a.cmax = 1;
  for (int j = 0; j < njob; ++j) {
    a.dot[j] = dot[j];
    a.dot[j].rc = dot_rows_per_chunk(dot[j].dim, dim_total, a.lgroups);
    a.dot[j].nchunk = (int)ceil_div(dot[j].dim, a.dot[j].rc);
    a.cmax = std::max<int64_t>(a.cmax, a.dot[j].nchunk);
    rc_max = std::max(rc_max, a.dot[j].rc);
    a.exp[j] = exp[j];
    dot_blocks += a.dot[j].nchunk * a.lgroups;
    exp_blocks += (int)ceil_div(exp[j].dim, kExpRows);
  }
  VSIE_REQUIRE((int64_t)njob * a.k * a.cmax <= (int64_t)h->part.n, VSIE_ERR_STATE, "farnear: partials too small");
  static bool attr = false;
  if (!attr) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_lr_dot, cudaFuncAttributeMaxDynamicSharedMemorySize, kRCMax * 16));
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_lr_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 16));
    attr = true;
  }
  launch_pdl(k_lr_dot, dim3(dot_blocks), dim3(256), (size_t)rc_max * sizeof(cplx), st, a);
  VSIE_CHECK_LAUNCH();
  launch_pdl(k_lr_expand, dim3(exp_blocks), dim3(256), (size_t)h->rank * sizeof(cplx), st, a);
  VSIE_CHECK_LAUNCH();
}

void zero(void* y, int64_t n, cudaStream_t st) {
  if (n > 0) VSIE_CHECK_CUDA(cudaMemsetAsync(y, 0, n * sizeof(cplx), st));
}

}  // namespace

void farnear_apply(vsie_farnear_s* h, const void* x, void* y, int op, int nrhs, cudaStream_t st) {
  VSIE_REQUIRE(op == VSIE_OP_N || op == VSIE_OP_T || op == VSIE_OP_C, VSIE_ERR_ARG, "op must be N, T or C");
  VSIE_REQUIRE(nrhs >= 1 && x && y, VSIE_ERR_ARG, "apply: bad arguments");
  const bool fwd = op == VSIE_OP_N;
  const int64_t din = fwd ? h->mf : h->mn, dout = fwd ? h->mn : h->mf;
  h->apply_calls++;
  if (h->rank == 0) return zero(y, dout * nrhs, st);
  const cplx* D = fwd ? h->W.p : h->U.p;   // the factor dotted with x
  const cplx* E = fwd ? h->U.p : h->W.p;   // the factor expanded into y
  const int cj = op == VSIE_OP_C;
  if (nrhs == 1) {
    LrJob dj{D, din, static_cast<const cplx*>(x), nullptr, cj, 0};
    LrJob ej{E, dout, nullptr, static_cast<cplx*>(y), cj, 0};
    lr_launch(h, 1, &dj, &ej, st);
    return;
  }
  // block RHS on the DMMA ZGEMM: T = D^T X (op C: on conj(X), then Y = E T conjugated back)
  const int k = h->rank;
  if (h->ws_nrhs < nrhs) {
    h->gemm_ws.alloc((size_t)64 * std::max<int64_t>(k, 1) * nrhs + (size_t)k * nrhs);
    h->xc.alloc((size_t)std::max(h->mn, h->mf) * nrhs);
    h->ws_nrhs = nrhs;
  }
  cplx* T = h->gemm_ws.p;
  cplx* ws = h->gemm_ws.p + (size_t)k * nrhs;
  const int64_t ws_elems = (int64_t)64 * k * nrhs;
  const cplx* X = static_cast<const cplx*>(x);
  if (cj) {
    launch_copy_conj(X, din, din, nrhs, h->xc.p, st);
    X = h->xc.p;
  }
  Zgemm g1;
  g1.ta = kT;
  g1.M[0] = k;
  g1.N[0] = nrhs;
  g1.K[0] = din;
  g1.A[0] = D;
  g1.lda[0] = din;
  g1.B[0] = X;
  g1.ldb[0] = din;
  g1.C[0] = T;
  g1.ldc[0] = k;
  launch_zgemm_dmma(g1, ws, ws_elems, st);
  Zgemm g2;
  g2.ta = kN;
  g2.M[0] = dout;
  g2.N[0] = nrhs;
  g2.K[0] = k;
  g2.A[0] = E;
  g2.lda[0] = dout;
  g2.B[0] = T;
  g2.ldb[0] = k;
  g2.C[0] = static_cast<cplx*>(y);
  g2.ldc[0] = dout;
  launch_zgemm_dmma(g2, ws, ws_elems, st);
  if (cj) launch_conj(static_cast<cplx*>(y), dout * nrhs, st);
}

void farnear_apply_pair(vsie_farnear_s* h, const void* x_far, void* y_near, const void* x_near, void* y_far,
                        cudaStream_t st) {
  VSIE_REQUIRE(x_far && y_near && x_near && y_far, VSIE_ERR_ARG, "apply_pair: NULL pointer");
  h->apply_calls++;
  if (h->rank == 0) {
    zero(y_near, h->mn, st);
    zero(y_far, h->mf, st);
    return;
  }
  LrJob d[2] = {{h->W.p, h->mf, static_cast<const cplx*>(x_far), nullptr, 0, 0},
                {h->U.p, h->mn, static_cast<const cplx*>(x_near), nullptr, 0, 0}};
  LrJob e[2] = {{h->U.p, h->mn, nullptr, static_cast<cplx*>(y_near), 0, 0},
                {h->W.p, h->mf, nullptr, static_cast<cplx*>(y_far), 0, 0}};
  lr_launch(h, 2, d, e, st);
}

}  // namespace vsie
