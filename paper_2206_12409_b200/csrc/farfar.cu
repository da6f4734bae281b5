// The dense far-far conductor block Z_cc^ff of the hybrid VSIE (PAPER.md
// P:159, Eq. 11 / 15; the EFIE of Eq. 1, on RWG functions).  Contract and
// entry definition: include/vsie_farfar.h (readings R-FF1..R-FF3).
//
// Kernels:
//  * ff_entry: the mixed-potential Galerkin entry of an RWG pair, summed over its 2 x 2 triangle
//    pairs -- regular pairs by the 3 x 3 rule (9 sincos), near pairs by the closed-form 1/R
//    potentials of a flat triangle at the 3 test nodes (both ways, symmetrised) plus the 3 x 3
//    rule on the bounded remainder (exp(-i k0 R) - 1) / (4 pi R).  FP64.
//  * k_ff_fill: one thread per stored element of the 128 x 128 lower-triangle tiles (the
//    symmetric half of the matrix: 8 x 10^8 entries at cfg 4, 12.8 GB).
//  * k_ff_tiles + k_ff_sum: the symmetric GEMV.  Z is HBM-bound (AI 0.5 flop/B), so each stored
//    tile is read ONCE for both of its products, Z_IJ x_J (rows) and Z_IJ^T x_I (columns): one
//    warp per tile, lane the rows lane + 32 q (4 coalesced 512-B segments per column), 4 columns
//    in flight, the column sums reduced across the warp by shuffles, no block barrier.  Per-tile
//    partials ([tile][2 x 128]) are summed per output block in a fixed order by k_ff_sum
//    (bitwise reproducible).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "farfar.hpp"
#include "geometry.hpp"

namespace vsie {

namespace {

constexpr int kTile = 128;
constexpr int kTriStride = 32;
constexpr double kInv4Pi = 0.079577471545947667884;

struct FfGeom {
  const double* tri;   // [nt][32]: V[0..8], c[9..11], n[12..14], q[15..23], A[24], L[25]
  const int* rt;       // [m][2]
  const double* rp;    // [m][8]
  int64_t m;
  double k0, scale_re, scale_im;
};

// closed-form I0 = int_T 1/R dS' and I1 = int_T (r' - r)/R dS' (oracle/farfar.py tri_potentials)
__device__ void tri_potentials(const double* __restrict__ T, double rx, double ry, double rz, double& I0,
                               double (&I1)[3]) {
  const double nx = T[12], ny = T[13], nz = T[14];
  const double h = (rx - T[0]) * nx + (ry - T[1]) * ny + (rz - T[2]) * nz;
  const double px = rx - h * nx, py = ry - h * ny, pz = rz - h * nz;
  const double ah = fabs(h);
  double i0 = 0, ix = 0, iy = 0, iz = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3;
    const double ax = T[3 * i], ay = T[3 * i + 1], az = T[3 * i + 2];
    const double bx = T[3 * j], by = T[3 * j + 1], bz = T[3 * j + 2];
    const double ex = bx - ax, ey = by - ay, ez = bz - az;
    const double el = sqrt(ex * ex + ey * ey + ez * ez);
    const double tx = ex / el, ty = ey / el, tz = ez / el;
    const double ux = ty * nz - tz * ny, uy = tz * nx - tx * nz, uz = tx * ny - ty * nx;
    const double lp = (bx - px) * tx + (by - py) * ty + (bz - pz) * tz;
    const double lm = (ax - px) * tx + (ay - py) * ty + (az - pz) * tz;
    const double P0 = (ax - px) * ux + (ay - py) * uy + (az - pz) * uz;
    const double R02 = P0 * P0 + h * h;
    const double Rp = sqrt(R02 + lp * lp), Rm = sqrt(R02 + lm * lm);
    double lg = 0, at = 0;
    if (R02 > (1e-14 * el) * (1e-14 * el)) {
      lg = log((Rp + lp) / (Rm + lm));
      at = atan(P0 * lp / (R02 + ah * Rp)) - atan(P0 * lm / (R02 + ah * Rm));
    }
    i0 += P0 * lg - ah * at;
    const double c = 0.5 * (R02 * lg + lp * Rp - lm * Rm);
    ix += c * ux;
    iy += c * uy;
    iz += c * uz;
  }
  I0 = i0;
  I1[0] = ix - h * i0 * nx;
  I1[1] = iy - h * i0 * ny;
  I1[2] = iz - h * i0 * nz;
}

// sum_q (A_a/3) int_{T_b} [(r_q - p_a).(r' - p_b) - 4/k0^2] g dS', singular part analytic
__device__ cplx k_near_oneway(const double* __restrict__ Ta, const double* pa, const double* __restrict__ Tb,
                              const double* pb, double k0) {
  const double c4 = 4.0 / (k0 * k0);
  double sr = 0, si = 0;
  for (int q = 0; q < 3; ++q) {
    const double rx = Ta[15 + 3 * q], ry = Ta[16 + 3 * q], rz = Ta[17 + 3 * q];
    double I0, I1[3];
    tri_potentials(Tb, rx, ry, rz, I0, I1);
    const double dx = rx - pa[0], dy = ry - pa[1], dz = rz - pa[2];
    const double sing = (dx * (I1[0] + (rx - pb[0]) * I0) + dy * (I1[1] + (ry - pb[1]) * I0) +
                         dz * (I1[2] + (rz - pb[2]) * I0) - c4 * I0) * kInv4Pi;
    double mr = 0, mi = 0;
    for (int s = 0; s < 3; ++s) {
      const double sx = Tb[15 + 3 * s], sy = Tb[16 + 3 * s], sz = Tb[17 + 3 * s];
      const double Rx = rx - sx, Ry = ry - sy, Rz = rz - sz;
      const double R = sqrt(Rx * Rx + Ry * Ry + Rz * Rz);
      const double f = dx * (sx - pb[0]) + dy * (sy - pb[1]) + dz * (sz - pb[2]) - c4;
      double gr, gi;
      if (R > 0) {
        double sn, cs;
        sincos(k0 * R, &sn, &cs);
        gr = (cs - 1.0) * kInv4Pi / R;
        gi = -sn * kInv4Pi / R;
      } else {
        gr = 0;
        gi = -k0 * kInv4Pi;
      }
      mr += f * gr;
      mi += f * gi;
    }
    sr += sing + Tb[24] / 3 * mr;
    si += Tb[24] / 3 * mi;
  }
  return cmk(Ta[24] / 3 * sr, Ta[24] / 3 * si);
}

__device__ cplx k_regular(const double* __restrict__ Ta, const double* pa, const double* __restrict__ Tb,
                          const double* pb, double k0) {
  const double c4 = 4.0 / (k0 * k0);
  double ar = 0, ai = 0;
  for (int q = 0; q < 3; ++q) {
    const double rx = Ta[15 + 3 * q], ry = Ta[16 + 3 * q], rz = Ta[17 + 3 * q];
    const double dx = rx - pa[0], dy = ry - pa[1], dz = rz - pa[2];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double sx = Tb[15 + 3 * s], sy = Tb[16 + 3 * s], sz = Tb[17 + 3 * s];
      const double Rx = rx - sx, Ry = ry - sy, Rz = rz - sz;
      const double r2 = Rx * Rx + Ry * Ry + Rz * Rz;
      const double ir = rsqrt(r2);
      double sn, cs;
      sincos(k0 * (r2 * ir), &sn, &cs);
      const double f = (dx * (sx - pb[0]) + dy * (sy - pb[1]) + dz * (sz - pb[2]) - c4) * ir;
      ar = fma(f, cs, ar);
      ai = fma(-f, sn, ai);
    }
  }
  const double w = Ta[24] / 3 * (Tb[24] / 3) * kInv4Pi;
  return cmk(w * ar, w * ai);
}

__device__ __forceinline__ bool tri_near(const double* Ta, const double* Tb) {
  const double dx = Ta[9] - Tb[9], dy = Ta[10] - Tb[10], dz = Ta[11] - Tb[11];
  const double L = 2.0 * fmax(Ta[25], Tb[25]);
  return dx * dx + dy * dy + dz * dz < L * L;
}

// Z[m, n] evaluated at (max, min)
__device__ cplx ff_entry(const FfGeom& g, int64_t r, int64_t c, int* near_count) {
  const int64_t m = r > c ? r : c, n = r > c ? c : r;
  const double lm = g.rp[8 * m + 6], ln = g.rp[8 * n + 6];
  double tr = 0, ti = 0;
  for (int sa = 0; sa < 2; ++sa) {
    const double* Ta = g.tri + (int64_t)kTriStride * g.rt[2 * m + sa];
    const double* pa = g.rp + 8 * m + 3 * sa;
    for (int sb = 0; sb < 2; ++sb) {
      const double* Tb = g.tri + (int64_t)kTriStride * g.rt[2 * n + sb];
      const double* pb = g.rp + 8 * n + 3 * sb;
      const double coef = ((sa == sb) ? 1.0 : -1.0) * lm * ln / (4.0 * Ta[24] * Tb[24]);
      cplx K;
      if (tri_near(Ta, Tb)) {
        const cplx k1 = k_near_oneway(Ta, pa, Tb, pb, g.k0), k2 = k_near_oneway(Tb, pb, Ta, pa, g.k0);
        K = cmk(0.5 * (k1.x + k2.x), 0.5 * (k1.y + k2.y));
        if (near_count) ++*near_count;
      } else {
        K = k_regular(Ta, pa, Tb, pb, g.k0);
      }
      tr += coef * K.x;
      ti += coef * K.y;
    }
  }
  return cmk(g.scale_re * tr - g.scale_im * ti, g.scale_re * ti + g.scale_im * tr);
}

__device__ __forceinline__ void tile_ij(int64_t t, int& I, int& J) {
  int64_t a = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) / 2.0);
  while (a * (a + 1) / 2 > t) --a;
  while ((a + 1) * (a + 2) / 2 <= t) ++a;
  I = (int)a;
  J = (int)(t - a * (a + 1) / 2);
}

__global__ void __launch_bounds__(256) k_ff_fill(FfGeom g, int64_t tiles, cplx* __restrict__ Z,
                                                 unsigned long long* near_pairs) {
  const int64_t total = tiles * kTile * kTile;
  int nc = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / (kTile * kTile);
    const int w = (int)(e - t * kTile * kTile);
    int I, J;
    tile_ij(t, I, J);
    const int64_t r = (int64_t)I * kTile + (w % kTile), c = (int64_t)J * kTile + (w / kTile);
    cplx v = cmk(0, 0);
    if (r < g.m && c < g.m) v = ff_entry(g, r, c, r >= c ? &nc : nullptr);
    Z[e] = v;
  }
  for (int o = 16; o > 0; o >>= 1) nc += __shfl_xor_sync(0xffffffffu, nc, o);
  if ((threadIdx.x & 31) == 0 && nc) atomicAdd(near_pairs, (unsigned long long)nc);
}

__global__ void __launch_bounds__(256) k_ff_list(FfGeom g, const int64_t* __restrict__ idx, int64_t count,
                                                 cplx* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = ff_entry(g, idx[2 * t], idx[2 * t + 1], nullptr);
}

__device__ __forceinline__ cplx opz(cplx v, int conj) { return conj ? cconj(v) : v; }

// per stored tile (I, J): part[t][0..128) = Z_IJ x_J, part[t][128..256) = Z_IJ^T x_I (I > J).
// One WARP per tile (no block barriers): lane holds rows lane + 32 q (q < 4) of the row sums;
// for each column j the 4 elements are coalesced 512-B segments, the column sum is a warp
// shuffle reduction.  Columns are unrolled by 4 (16 independent 16-B loads per lane in flight).
__global__ void __launch_bounds__(256) k_ff_tiles(const cplx* __restrict__ Z, int64_t tiles, int64_t m,
                                                  const cplx* __restrict__ x, int conj, cplx* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  pdl_wait();
  for (int64_t t = warp; t < tiles; t += nwarps) {
    int I, J;
    tile_ij(t, I, J);
    const int64_t i0 = (int64_t)I * kTile, j0 = (int64_t)J * kTile;
    cplx xi[4], acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t r = i0 + lane + 32 * q;
      xi[q] = r < m ? x[r] : cmk(0, 0);
      acc[q] = cmk(0, 0);
    }
    const bool offdiag = I != J;
    const cplx* Zt = Z + t * kTile * kTile + lane;
    cplx* pt = part + t * 2 * kTile;
    for (int j = 0; j < kTile; j += 4) {
      cplx z[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) z[c][q] = opz(__ldcs(Zt + (int64_t)kTile * (j + c) + 32 * q), conj);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t cj = j0 + j + c;
        const cplx xj = cj < m ? x[cj] : cmk(0, 0);
        cplx cs = cmk(0, 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          cfma(acc[q], z[c][q], xj);
          cfma(cs, z[c][q], xi[q]);
        }
        if (offdiag) {
          for (int o = 16; o > 0; o >>= 1) {
            cs.x += __shfl_xor_sync(0xffffffffu, cs.x, o);
            cs.y += __shfl_xor_sync(0xffffffffu, cs.y, o);
          }
          if (lane == 0) pt[kTile + j + c] = cs;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) pt[lane + 32 * q] = acc[q];
  }
  pdl_trigger();
}

// y[r] = (acc ? y[r] : 0) + sum_{J <= I} part[(I, J)].N[r'] + sum_{K > I} part[(K, I)].T[r'],
// r = 128 I + r', in that order
__global__ void __launch_bounds__(kTile) k_ff_sum(const cplx* __restrict__ part, int nb, int64_t m, cplx* y,
                                                  int accumulate) {
  const int I = blockIdx.x, rl = threadIdx.x;
  const int64_t r = (int64_t)I * kTile + rl;
  pdl_wait();
  if (r >= m) return;
  cplx s0 = cmk(0, 0), s1 = cmk(0, 0);
  const int64_t base = (int64_t)I * (I + 1) / 2;
  int J = 0;
  for (; J + 1 <= I; J += 2) {
    s0 = cadd(s0, __ldcg(part + (base + J) * 2 * kTile + rl));
    s1 = cadd(s1, __ldcg(part + (base + J + 1) * 2 * kTile + rl));
  }
  if (J <= I) s0 = cadd(s0, __ldcg(part + (base + J) * 2 * kTile + rl));
  for (int K = I + 1; K < nb; ++K) s1 = cadd(s1, __ldcg(part + ((int64_t)K * (K + 1) / 2 + I) * 2 * kTile + kTile + rl));
  cplx v = cadd(s0, s1);
  if (accumulate) v = cadd(v, y[r]);
  y[r] = v;
}

FfGeom geom_of(const vsie_farfar_s* h) {
  FfGeom g;
  g.tri = h->tri.p;
  g.rt = h->rt.p;
  g.rp = h->rp.p;
  g.m = h->m;
  g.k0 = h->k0;
  g.scale_re = h->scale_re;
  g.scale_im = h->scale_im;
  return g;
}

}  // namespace

void farfar_build(const vsie_mesh* meshes, int n_meshes, double freq, double scale_re, double scale_im, int device,
                  vsie_farfar_s* h) {
  const auto t0 = std::chrono::steady_clock::now();
  VSIE_REQUIRE(meshes != nullptr && n_meshes >= 1, VSIE_ERR_ARG, "farfar_build: no meshes");
  VSIE_REQUIRE(freq > 0 && std::isfinite(freq), VSIE_ERR_ARG, "freq must be > 0");
  VSIE_REQUIRE(std::isfinite(scale_re) && std::isfinite(scale_im), VSIE_ERR_ARG, "bad scale");
  // host tables: triangles of every mesh (global ids), RWG functions in canonical order
  std::vector<double> tri;
  std::vector<int> rt;
  std::vector<double> rp;
  int64_t tri_base = 0;
  for (int k = 0; k < n_meshes; ++k) {
    const vsie_mesh& ms = meshes[k];
    const std::vector<RwgRec> rw = extract_rwgs(ms);   // validates the mesh
    const double* X = ms.xyz;
    const int32_t* T = ms.tri;
    for (int64_t t = 0; t < ms.n_triangles; ++t) {
      double rec[kTriStride] = {0};
      double* V = rec;
      for (int v = 0; v < 3; ++v)
        for (int c = 0; c < 3; ++c) V[3 * v + c] = X[3 * T[3 * t + v] + c];
      const double e1[3] = {V[3] - V[0], V[4] - V[1], V[5] - V[2]};
      const double e2[3] = {V[6] - V[0], V[7] - V[1], V[8] - V[2]};
      const double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
      const double cn = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
      double L = 0;
      for (int e = 0; e < 3; ++e) {
        const int f = (e + 1) % 3;
        double d2 = 0;
        for (int c = 0; c < 3; ++c) d2 += (V[3 * f + c] - V[3 * e + c]) * (V[3 * f + c] - V[3 * e + c]);
        L = std::max(L, std::sqrt(d2));
      }
      for (int c = 0; c < 3; ++c) {
        rec[9 + c] = (V[c] + V[3 + c] + V[6 + c]) / 3.0;
        rec[12 + c] = cr[c] / cn;
      }
      for (int q = 0; q < 3; ++q)
        for (int c = 0; c < 3; ++c) {
          const double w0 = q == 0 ? 2.0 / 3.0 : 1.0 / 6.0, w1 = q == 1 ? 2.0 / 3.0 : 1.0 / 6.0,
                       w2 = q == 2 ? 2.0 / 3.0 : 1.0 / 6.0;
          rec[15 + 3 * q + c] = w0 * V[c] + w1 * V[3 + c] + w2 * V[6 + c];
        }
      rec[24] = 0.5 * cn;
      rec[25] = L;
      tri.insert(tri.end(), rec, rec + kTriStride);
    }
    for (const RwgRec& r : rw) {
      rt.push_back((int)(tri_base + r.tp));
      rt.push_back((int)(tri_base + r.tm));
      double rec[8] = {0};
      for (int c = 0; c < 3; ++c) {
        rec[c] = X[3 * r.pp + c];
        rec[3 + c] = X[3 * r.pm + c];
      }
      double l2 = 0;
      for (int c = 0; c < 3; ++c) l2 += (X[3 * r.a + c] - X[3 * r.b + c]) * (X[3 * r.a + c] - X[3 * r.b + c]);
      rec[6] = std::sqrt(l2);
      rp.insert(rp.end(), rec, rec + 8);
    }
    tri_base += ms.n_triangles;
  }
  h->m = (int64_t)rt.size() / 2;
  h->nt = tri_base;
  VSIE_REQUIRE(h->m >= 1, VSIE_ERR_GEOMETRY, "meshes have no interior edge (no RWG function)");
  VSIE_REQUIRE(tri_base < INT32_MAX, VSIE_ERR_ARG, "too many triangles");
  if (device >= 0) VSIE_CHECK_CUDA(cudaSetDevice(device));
  VSIE_CHECK_CUDA(cudaGetDevice(&h->device));
  h->k0 = 2.0 * 3.14159265358979323846 * freq / 299792458.0;
  h->scale_re = scale_re;
  h->scale_im = scale_im;
  h->nb = (int)ceil_div(h->m, kTile);
  h->tiles = (int64_t)h->nb * (h->nb + 1) / 2;
  h->tri.alloc(tri.size());
  h->rt.alloc(rt.size());
  h->rp.alloc(rp.size());
  VSIE_CHECK_CUDA(cudaMemcpy(h->tri.p, tri.data(), tri.size() * sizeof(double), cudaMemcpyHostToDevice));
  VSIE_CHECK_CUDA(cudaMemcpy(h->rt.p, rt.data(), rt.size() * sizeof(int), cudaMemcpyHostToDevice));
  VSIE_CHECK_CUDA(cudaMemcpy(h->rp.p, rp.data(), rp.size() * sizeof(double), cudaMemcpyHostToDevice));
  h->Z.alloc((size_t)h->tiles * kTile * kTile);
  h->part.alloc((size_t)h->tiles * 2 * kTile);
  DevBuf<unsigned long long> nearc(1);
  VSIE_CHECK_CUDA(cudaMemset(nearc.p, 0, sizeof(unsigned long long)));
  const int64_t total = h->tiles * kTile * kTile;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 64);
  k_ff_fill<<<blocks, 256>>>(geom_of(h), h->tiles, h->Z.p, nearc.p);
  VSIE_CHECK_LAUNCH();
  unsigned long long nc = 0;
  VSIE_CHECK_CUDA(cudaMemcpy(&nc, nearc.p, sizeof(nc), cudaMemcpyDeviceToHost));
  h->near_pairs = (int64_t)nc;
  VSIE_CHECK_CUDA(cudaDeviceSynchronize());
  h->build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void farfar_entries(vsie_farfar_s* h, const int64_t* idx, int64_t count, void* out, cudaStream_t st) {
  VSIE_REQUIRE(count >= 0 && (count == 0 || (idx && out)), VSIE_ERR_ARG, "entries: bad arguments");
  if (count == 0) return;
  const int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 32);
  k_ff_list<<<blocks, 256, 0, st>>>(geom_of(h), idx, count, static_cast<cplx*>(out));
  VSIE_CHECK_LAUNCH();
}

void farfar_apply(vsie_farfar_s* h, const void* x, void* y, int op, int nrhs, bool accumulate, cudaStream_t st) {
  VSIE_REQUIRE(op == VSIE_OP_N || op == VSIE_OP_T || op == VSIE_OP_C, VSIE_ERR_ARG, "op must be N, T or C");
  VSIE_REQUIRE(nrhs >= 1 && x && y, VSIE_ERR_ARG, "apply: bad arguments");
  h->apply_calls++;
  int dev = 0, nsm = 0, per = 0;
  VSIE_CHECK_CUDA(cudaGetDevice(&dev));
  VSIE_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ff_tiles, 256, 0));
  const int grid = (int)std::min<int64_t>(h->tiles, (int64_t)nsm * std::max(per, 1));
  for (int r = 0; r < nrhs; ++r) {
    const cplx* xr = static_cast<const cplx*>(x) + (int64_t)r * h->m;
    cplx* yr = static_cast<cplx*>(y) + (int64_t)r * h->m;
    // OP_C: conj(Z) x = conj(Z conj(x)) -- here conj applied to each loaded element
    launch_pdl(k_ff_tiles, dim3(grid), dim3(256), 0, st, (const cplx*)h->Z.p, h->tiles, h->m, xr,
               op == VSIE_OP_C ? 1 : 0, h->part.p);
    VSIE_CHECK_LAUNCH();
    launch_pdl(k_ff_sum, dim3(h->nb), dim3(kTile), 0, st, (const cplx*)h->part.p, h->nb, h->m, yr,
               accumulate ? 1 : 0);
    VSIE_CHECK_LAUNCH();
  }
}

void farfar_export(vsie_farfar_s* h, void* host_dense) {
  VSIE_REQUIRE(host_dense != nullptr, VSIE_ERR_ARG, "export: NULL");
  VSIE_CHECK_CUDA(cudaDeviceSynchronize());
  std::vector<cplx> tiles((size_t)h->tiles * kTile * kTile);
  VSIE_CHECK_CUDA(cudaMemcpy(tiles.data(), h->Z.p, tiles.size() * sizeof(cplx), cudaMemcpyDeviceToHost));
  cplx* D = static_cast<cplx*>(host_dense);
  const int64_t m = h->m;
  for (int I = 0; I < h->nb; ++I)
    for (int J = 0; J <= I; ++J) {
      const cplx* t = tiles.data() + ((int64_t)I * (I + 1) / 2 + J) * kTile * kTile;
      for (int j = 0; j < kTile; ++j)
        for (int i = 0; i < kTile; ++i) {
          const int64_t r = (int64_t)I * kTile + i, c = (int64_t)J * kTile + j;
          if (r >= m || c >= m) continue;
          D[r + m * c] = t[i + kTile * j];
          D[c + m * r] = t[i + kTile * j];
        }
    }
}

}  // namespace vsie
