// Z_bc entry evaluation: the black-box entry function of the
// TT-cross — the 5-D surface-volume integral of
// the dyadic Green's function (Eq. 3) between a PWC voxel testing
// function and an RWG basis function, by the fixed non-singular
// quadrature of SURVEY §8c-E (2x2x2 Gauss per voxel x 3-point rule per
// triangle, 48 pair interactions per entry; or the paper's far-block rule of P:287, one
// voxel point x one point per triangle, 2 pairs per entry, build option quad_rule = 1).
//
// Per pair, with R = r_p - r_s, u = 1/(k0 |R|), g = exp(-i k0 |R|)/(4 pi |R|):
//   [G(R) J]_chi = g [ alpha J_chi + beta Rhat_chi (Rhat . J) ],
//   alpha = 1 - i u - u^2,  beta = -1 + 3 i u + 3 u^2.
// FP64 throughout (one rsqrt, one sincos per pair); FMA contraction on.
#include "kernels.cuh"

#include <cmath>

namespace vsie {

namespace {

// Accumulates sum_{p, s} pw_p [G(r_p - r_s) J_s]_chi (without w, scale); pw_p = 1/(4 pi)
// times the PWL test function at node p (1 for PWC testing, +-1/(2 sqrt 3) for a linear one)
// for one voxel centre (cx, cy, cz) and one RWG source record s36.
//
// chi is a run-time value selected inside one instruction stream (a warp of list-mode
// entries holds all three components: templated bodies would run all three).
//
// Phase: the 8 voxel nodes of a source node s sit within |d| = |h| / (2 sqrt 3) of the voxel
// centre, so with R0 = |c - r_s|, k0 R_p = k0 R0 + delta_p, |delta_p| <= k0 |d| (<= 0.016 rad at
// the 5 mm voxels of cfg 1).  One sincos(k0 R0) per source node and the order-7 Taylor
// polynomials of cos / sin(delta_p) (truncation <= |delta|^8 / 8! < 1e-19) per pair give
// exp(-i k0 R_p) by angle addition -- the same value as a sincos per pair to rounding, at
// ~1/3 of its FP64 instructions (g.taylor; otherwise a sincos per pair).
template <int NP, bool SM>
__device__ __forceinline__ void entry_acc(const EntryGeom& g, int chi, double cx, double cy, double cz,
                                          const double* __restrict__ s36, double& ar, double& ai) {
  // SM: the source record is staged in shared memory (block mode); else read through L1 as
  // three 16-B loads per source node (list mode: 32 different records per warp, so the load
  // instruction count, not the bytes, is what the LSU pays for)
#pragma unroll 1
  for (int q = 0; q < g.nsrc; ++q) {
    double2 a, b, c;
    if (SM) {
      a = make_double2(s36[6 * q], s36[6 * q + 1]);
      b = make_double2(s36[6 * q + 2], s36[6 * q + 3]);
      c = make_double2(s36[6 * q + 4], s36[6 * q + 5]);
    } else {
      const double2* p2 = reinterpret_cast<const double2*>(s36 + 6 * q);
      a = __ldg(p2);
      b = __ldg(p2 + 1);
      c = __ldg(p2 + 2);
    }
    const double sx = a.x, sy = a.y, sz = b.x;
    const double jx = b.y, jy = c.x, jz = c.y;
    const double jc = chi == 0 ? jx : (chi == 1 ? jy : jz);
    const double bx = cx - sx, by = cy - sy, bz = cz - sz;
    double s0 = 0, c0 = 1, kr0 = 0;
    if (g.taylor) {
      const double b2 = fma(bx, bx, fma(by, by, bz * bz));
      kr0 = g.k0 * (b2 * rsqrt(b2));
      sincos(kr0, &s0, &c0);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      // NP = 8: the 2 x 2 x 2 Gauss nodes c +- h / (2 sqrt 3); NP = 1: the centre
      const double rx = NP == 1 ? bx : ((p & 1) ? bx + g.dx : bx - g.dx);
      const double ry = NP == 1 ? by : ((p & 2) ? by + g.dy : by - g.dy);
      const double rz = NP == 1 ? bz : ((p & 4) ? bz + g.dz : bz - g.dz);
      const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
      const double ir = rsqrt(r2);
      const double R = r2 * ir;
      double sn, cs;
      if (g.taylor) {
        const double dl = fma(g.k0, R, -kr0), d2 = dl * dl;
        // cos dl = 1 - d2/2 + d2^2/24 - d2^3/720,  sin dl = dl (1 - d2/6 + d2^2/120 - d2^3/5040)
        const double cd = fma(d2, fma(d2, fma(d2, -1.0 / 720.0, 1.0 / 24.0), -0.5), 1.0);
        const double sd = dl * fma(d2, fma(d2, fma(d2, -1.0 / 5040.0, 1.0 / 120.0), -1.0 / 6.0), 1.0);
        cs = fma(c0, cd, -s0 * sd);
        sn = fma(s0, cd, c0 * sd);
      } else {
        sincos(g.k0 * R, &sn, &cs);
      }
      const double u = g.inv_k0 * ir;
      const double u2 = u * u;
      const double rc = chi == 0 ? rx : (chi == 1 ? ry : rz);
      const double rj = fma(rx, jx, fma(ry, jy, rz * jz));
      const double t = rj * rc * (ir * ir);                 // Rhat_chi (Rhat . J)
      const double A = fma(1.0 - u2, jc, (3.0 * u2 - 1.0) * t);  // Re(alpha J_chi + beta t)
      const double B = u * (3.0 * t - jc);                       // Im(...)
      const double qq = ir * g.pw[p];
      // g * (A + iB) = qq (cs - i sn)(A + i B)
      ar = fma(qq, fma(cs, A, sn * B), ar);
      ai = fma(qq, fma(cs, B, -sn * A), ai);
    }
  }
}

template <bool SM>
__device__ __forceinline__ cplx entry_value(const EntryGeom& g, int chi, int i1, int i2, int i3,
                                            const double* __restrict__ s36) {
  const double cx = g.ox + i1 * g.hx, cy = g.oy + i2 * g.hy, cz = g.oz + i3 * g.hz;
  double ar = 0, ai = 0;
  if (g.nodes == 1)
    entry_acc<1, SM>(g, chi, cx, cy, cz, s36, ar, ai);
  else
    entry_acc<8, SM>(g, chi, cx, cy, cz, s36, ar, ai);
  ar *= g.w;
  ai *= g.w;
  return cmk(g.scale_re * ar - g.scale_im * ai, g.scale_re * ai + g.scale_im * ar);
}

__global__ void __launch_bounds__(256) k_entries_list(EntryGeom g, const int64_t* __restrict__ idx,
                                                      int64_t count, cplx* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx[2 * t], col = idx[2 * t + 1];
    const int chi = (int)(row / g.nv);
    const int64_t v = row - chi * g.nv;
    const int i1 = (int)(v % g.n1);
    const int i2 = (int)((v / g.n1) % g.n2);
    const int i3 = (int)(v / ((int64_t)g.n1 * g.n2));
    out[t] = entry_value<false>(g, chi, i1, i2, i3, g.src + 36 * col);
  }
}

// Block mode: tiles of 256 consecutive entries (rows fastest), so a tile touches only
// ceil(256 / rows) + 1 columns of the supercore: their RWG source records (the quadrature
// nodes and moments, 36 doubles each) are staged in shared memory once per tile.
constexpr int kEntThreads = 256;
constexpr int kEntPer = 4;                           // entries per thread and tile
constexpr int kEntTile = kEntThreads * kEntPer;
constexpr int kEntMaxCols = 96;   // rows >= 12 (every k_n of the configs); wider tiles fall back

__device__ __forceinline__ void block_coords(const BlockDesc& b, int64_t r, int64_t c, int& i1, int& i2, int& i3,
                                             int64_t& n) {
  const int64_t alpha = r % b.rl, ik = r / b.rl;
  const int64_t ik1 = c % b.nk1, beta = c / b.nk1;
  if (b.k == 1) {
    i1 = (int)ik;
    i2 = (int)ik1;
    i3 = b.right[2 * beta];
    n = b.right[2 * beta + 1];
  } else if (b.k == 2) {
    i1 = b.left[2 * alpha];
    i2 = (int)ik;
    i3 = (int)ik1;
    n = b.right[2 * beta];
  } else {
    i1 = b.left[2 * alpha];
    i2 = b.left[2 * alpha + 1];
    i3 = (int)ik;
    n = ik1;
  }
}

__global__ void __launch_bounds__(kEntThreads) k_entries_block(EntryGeom g, BlockDesc b, cplx* __restrict__ out) {
  __shared__ double rec[kEntMaxCols][36];
  const int64_t r0 = b.row1 > b.row0 ? b.row0 : 0;
  const int64_t rows = b.row1 > b.row0 ? b.row1 - b.row0 : b.rl * b.nk;   // rows evaluated
  const int64_t total = rows * (b.col1 - b.col0);
  const int64_t ntile = (total + kEntTile - 1) / kEntTile;
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int64_t t0 = tile * kEntTile;
    const int64_t cl0 = t0 / rows, cl1 = min(total - 1, t0 + kEntTile - 1) / rows;
    const int ncl = (int)(cl1 - cl0 + 1);
    __syncthreads();   // the previous tile's records are no longer read
    for (int e = threadIdx.x; e < ncl * 36; e += kEntThreads) {
      const int q = e / 36, w = e - 36 * q;
      int i1, i2, i3;
      int64_t n;
      block_coords(b, r0, b.col0 + cl0 + q, i1, i2, i3, n);
      rec[q][w] = __ldg(g.src + 36 * n + w);
    }
    __syncthreads();
#pragma unroll 1
    for (int u = 0; u < kEntPer; ++u) {
      const int64_t t = t0 + u * kEntThreads + threadIdx.x;
      if (t < total) {
        const int64_t rr = t % rows, cl = t / rows;
        int i1, i2, i3;
        int64_t n;
        block_coords(b, r0 + rr, b.col0 + cl, i1, i2, i3, n);
        out[rr + b.ld * cl] = entry_value<true>(g, b.chi, i1, i2, i3, rec[cl - cl0]);
      }
    }
  }
}

// the same without staging (tiles wider than kEntMaxCols columns: rows < 12)
__global__ void __launch_bounds__(256) k_entries_block_direct(EntryGeom g, BlockDesc b, cplx* __restrict__ out) {
  const int64_t r0 = b.row1 > b.row0 ? b.row0 : 0;
  const int64_t rows = b.row1 > b.row0 ? b.row1 - b.row0 : b.rl * b.nk;
  const int64_t total = rows * (b.col1 - b.col0);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = t % rows, cl = t / rows;
    int i1, i2, i3;
    int64_t n;
    block_coords(b, r0 + rr, b.col0 + cl, i1, i2, i3, n);
    out[rr + b.ld * cl] = entry_value<false>(g, b.chi, i1, i2, i3, g.src + 36 * n);
  }
}

int grid_for(int64_t work, int threads) {
  int64_t blocks = ceil_div(work, threads);
  const int64_t cap = 148 * 64;
  return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

}  // namespace

void launch_entries_list(const EntryGeom& g, const int64_t* idx, int64_t count, cplx* out,
                         cudaStream_t st) {
  if (count <= 0) return;
  k_entries_list<<<grid_for(count, 256), 256, 0, st>>>(g, idx, count, out);
  VSIE_CHECK_LAUNCH();
}

void launch_entries_block(const EntryGeom& g, const BlockDesc& b, cplx* out, cudaStream_t st) {
  const int64_t rows = b.row1 > b.row0 ? b.row1 - b.row0 : b.rl * b.nk;
  const int64_t total = rows * (b.col1 - b.col0);
  if (total <= 0) return;
  if (kEntTile / rows + 2 <= kEntMaxCols)
    k_entries_block<<<grid_for(ceil_div(total, kEntPer), kEntThreads), kEntThreads, 0, st>>>(g, b, out);
  else
    k_entries_block_direct<<<grid_for(total, 256), 256, 0, st>>>(g, b, out);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
