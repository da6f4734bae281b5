// Device kernels of the TT-cross driver (see crosskern.cuh).
//
// * one-sided Jacobi SVD (Hestenes): each launch performs one round of the
//   round-robin ordering, one CTA per column pair, complex rotation
//     a_i' = cs a_i - sn e^{-i phi} a_j,   a_j' = sn a_i + cs e^{-i phi} a_j,
//   with c = a_i^H a_j = |c| e^{i phi}, zeta = (|a_j|^2 - |a_i|^2) / (2|c|),
//   t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), cs = 1/sqrt(1 + t^2), sn = cs t;
// * maxvol: LU with partial pivoting for the initial rows,
//   B = A A[I]^{-1} = P^T [I; L2 L1^{-1}], then rank-1 updates
//   B <- B - B[:, j*] (B[i*, :] - e_j*^T) / B[i*, j*] while max |B| > 1 + tau,
//   ties broken towards the smallest (original row, column) as in the oracle.
#include "crosskern.cuh"

#include <cooperative_groups.h>

#include <algorithm>

namespace vsie {

namespace {

constexpr int NT = 256;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_gaussian(cplx* out, int64_t n, uint64_t seed) {
  const uint64_t s = splitmix64(seed);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = splitmix64(s ^ (2 * (uint64_t)e)), b = splitmix64(s ^ (2 * (uint64_t)e + 1));
    const double u1 = ((a >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = (b >> 11) * 0x1.0p-53;        // [0, 1)
    const double rr = sqrt(-2.0 * log(u1)) * 0.70710678118654752440;
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    out[e] = cmk(rr * cs, rr * sn);
  }
}

template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double* sh /* >= 8 * N */) {
#pragma unroll
  for (int k = 0; k < N; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) sh[w * N + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double s = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += sh[q * N + k];
    v[k] = s;
  }
}

// one Jacobi rotation of columns (i, j) of A (and V), by one CTA; returns 1 if rotated
__device__ int jacobi_pair(cplx* A, int64_t p, int64_t lda, cplx* V, int64_t q, int i, int j, double thr,
                           double small2, double* sh) {
  if (i >= q || j >= q) return 0;
  cplx* Ai = A + lda * i;
  cplx* Aj = A + lda * j;
  double v[4] = {0, 0, 0, 0};
  for (int64_t r = threadIdx.x; r < p; r += NT) {
    const cplx x = Ai[r], y = Aj[r];
    v[0] += x.x * x.x + x.y * x.y;
    v[1] += y.x * y.x + y.y * y.y;
    v[2] += x.x * y.x + x.y * y.y;  // Re(conj(x) y)
    v[3] += x.x * y.y - x.y * y.x;  // Im(conj(x) y)
  }
  block_sum<4>(v, sh);
  const double a = v[0], b = v[1];
  const double cabs = sqrt(v[2] * v[2] + v[3] * v[3]);
  // columns below the noise floor (||a||^2 <= small2) are treated as zero (as in
  // LAPACK xGESVJ): rotating them against large columns only re-injects rounding noise
  if (!(a > small2 && b > small2) || !(cabs > thr * sqrt(a) * sqrt(b))) return 0;
  const double zeta = (b - a) / (2.0 * cabs);
  const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
  const cplx ph = cmk(v[2] / cabs, -v[3] / cabs);  // e^{-i phi}
  const cplx snph = cmk(sn * ph.x, sn * ph.y), csph = cmk(cs * ph.x, cs * ph.y);
  for (int64_t r = threadIdx.x; r < p; r += NT) {
    const cplx x = Ai[r], y = Aj[r];
    const cplx py = cmul(snph, y), qy = cmul(csph, y);
    Ai[r] = cmk(cs * x.x - py.x, cs * x.y - py.y);
    Aj[r] = cmk(sn * x.x + qy.x, sn * x.y + qy.y);
  }
  if (V) {
    cplx* Vi = V + q * i;
    cplx* Vj = V + q * j;
    for (int64_t r = threadIdx.x; r < q; r += NT) {
      const cplx x = Vi[r], y = Vj[r];
      const cplx py = cmul(snph, y), qy = cmul(csph, y);
      Vi[r] = cmk(cs * x.x - py.x, cs * x.y - py.y);
      Vj[r] = cmk(sn * x.x + qy.x, sn * x.y + qy.y);
    }
  }
  return 1;
}

__global__ void __launch_bounds__(NT) k_jacobi_round(cplx* A, int64_t p, int64_t lda, cplx* V, int64_t q,
                                                     const int2* pairs, double thr, double small2, unsigned* cnt) {
  __shared__ double sh[8 * 4];
  const int2 pr = pairs[blockIdx.x];
  if (jacobi_pair(A, p, lda, V, q, pr.x, pr.y, thr, small2, sh) && threadIdx.x == 0) atomicAdd(cnt, 1u);
}

// All sweeps of a cyclic one-sided Jacobi in ONE cooperative launch: CTA k owns
// pair slot k of every round, rounds are separated by grid-wide barriers, and
// the sweep loop ends (uniformly) when a sweep applied no rotation.
// cnt[0..1]: alternating per-sweep rotation counters (zeroed by the host);
// cnt[2] receives the number of sweeps.
__global__ void __launch_bounds__(NT) k_jacobi_coop(cplx* A, int64_t p, int64_t lda, cplx* V, int64_t q,
                                                    const int2* pairs, int nrounds, double thr, double small2,
                                                    int max_sweeps, unsigned* cnt) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[8 * 4];
  const int half = gridDim.x;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    unsigned* mine = cnt + (sweep & 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(sweep + 1) & 1] = 0;
    for (int t = 0; t < nrounds; ++t) {
      const int2 pr = pairs[(int64_t)t * half + blockIdx.x];
      if (jacobi_pair(A, p, lda, V, q, pr.x, pr.y, thr, small2, sh) && threadIdx.x == 0) atomicAdd(mine, 1u);
      grid.sync();
    }
    const unsigned rot = *((volatile unsigned*)mine);
    if (rot == 0) break;
    grid.sync();  // everyone has read `mine` before it is zeroed in the next-but-one sweep
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[2] = (unsigned)(sweep + 1);
}

__global__ void __launch_bounds__(NT) k_col_norms(const cplx* A, int64_t p, int64_t lda, double* out) {
  const cplx* a = A + lda * blockIdx.x;
  double v[1] = {0};
  for (int64_t r = threadIdx.x; r < p; r += NT) v[0] += cabs2(a[r]);
  __shared__ double sh[8];
  block_sum<1>(v, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt(v[0]);
}

__global__ void __launch_bounds__(NT) k_frob_partial(const cplx* A, int64_t n, double* partial) {
  double v[1] = {0};
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < n; e += (int64_t)gridDim.x * NT) v[0] += cabs2(A[e]);
  __shared__ double sh[8];
  block_sum<1>(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v[0];
}
__global__ void k_frob_final(const double* partial, int np, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0;
    for (int i = 0; i < np; ++i) s += partial[i];
    *out = s;
  }
}

__global__ void k_gather_cols(const cplx* src, int64_t rows, int64_t lds, const int* idx, const double* scale,
                              int ncols, cplx* dst, int64_t ldd, int conj) {
  const int j = blockIdx.y;
  const cplx* s = src + lds * idx[j];
  const double f = scale ? scale[j] : 1.0;
  for (int64_t r = blockIdx.x * (int64_t)NT + threadIdx.x; r < rows; r += (int64_t)gridDim.x * NT) {
    cplx v = s[r];
    dst[r + ldd * j] = cmk(f * v.x, conj ? -f * v.y : f * v.y);
  }
}

__global__ void k_gather_rows(const cplx* src, int64_t lds, const int* idx, int nr, int64_t cols, cplx* dst) {
  const int64_t total = (int64_t)nr * cols;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
    const int64_t i = e % nr, c = e / nr;
    dst[e] = src[idx[i] + lds * c];
  }
}

__global__ void k_transpose(const cplx* src, int64_t R, int64_t C, cplx* dst, int conj) {
  __shared__ cplx tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows per pass
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + tx, c = c0 + k;
    if (r < R && c < C) tile[k][tx] = src[r + R * c];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t c = c0 + tx, r = r0 + k;
    if (r < R && c < C) {
      cplx v = tile[tx][k];
      if (conj) v.y = -v.y;
      dst[c + C * r] = v;
    }
  }
}

// ----------------------------------------------------------------------- argmax helpers
__device__ __forceinline__ bool better(double v, int64_t key, double bv, int64_t bkey) {
  return v > bv || (v == bv && key < bkey);
}

__device__ void block_argmax(ArgMax& m, ArgMax* sh /* >= 8 */) {
  for (int o = 16; o > 0; o >>= 1) {
    const double v = __shfl_xor_sync(0xffffffffu, m.v, o);
    const long long key = __shfl_xor_sync(0xffffffffu, (long long)m.key, o);
    const long long i = __shfl_xor_sync(0xffffffffu, (long long)m.i, o);
    const int c = __shfl_xor_sync(0xffffffffu, m.c, o);
    if (better(v, key, m.v, m.key)) { m.v = v; m.key = key; m.i = i; m.c = c; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (better(sh[q].v, sh[q].key, sh[0].v, sh[0].key)) sh[0] = sh[q];
  }
  __syncthreads();
  m = sh[0];
}

// Step j of the LU: scale column j below the diagonal (when scale), rank-1 update of columns
// (j, c1), then argmax partials of column j + 1 over rows > j (when j + 1 < r and argmax).
// The blocked LU (panel width kLuPanel) passes c1 = the panel end; the trailing columns are
// updated by a TRSM + ZGEMM per panel.
__global__ void __launch_bounds__(NT) k_lu_update(cplx* W, int64_t n, int r, int j, int c1, int scale, int argmax,
                                                  ArgMax* partials) {
  extern __shared__ cplx urow[];
  __shared__ cplx inv;
  __shared__ ArgMax sh[8];
  if (j >= 0 && scale) {
    for (int c = j + 1 + threadIdx.x; c < c1; c += NT) urow[c] = W[j + n * c];
    if (threadIdx.x == 0) {
      const cplx pv = W[j + n * j];
      const double d = cabs2(pv);
      inv = cmk(pv.x / d, -pv.y / d);
    }
    __syncthreads();
  }
  ArgMax best{-1.0, INT64_MAX, -1, j + 1};
  for (int64_t i = j + 1 + blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    if (j >= 0 && scale) {
      const cplx l = cmul(W[i + n * j], inv);
      W[i + n * j] = l;
      for (int c = j + 1; c < c1; ++c) {
        const cplx u = urow[c];
        cplx w = W[i + n * c];
        w.x -= l.x * u.x - l.y * u.y;
        w.y -= l.x * u.y + l.y * u.x;
        W[i + n * c] = w;
      }
    }
    if (argmax && j + 1 < r) {
      const double v = cabs2(W[i + n * (j + 1)]);
      if (better(v, i, best.v, best.key)) { best.v = v; best.key = i; best.i = i; }
    }
  }
  block_argmax(best, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = best;
}

// U12 = L11^{-1} A12 in place: L11 the unit lower jb x jb block at (j0, j0), A12 rows
// [j0, j0 + jb), columns [j0 + jb, r); one thread per column, L11 in smem
__global__ void __launch_bounds__(NT) k_lu_trsm(cplx* W, int64_t n, int r, int j0, int jb) {
  __shared__ cplx L[kLuPanel * kLuPanel];
  for (int e = threadIdx.x; e < jb * jb; e += NT) {
    const int i = e % jb, k = e / jb;
    L[e] = W[(j0 + i) + n * (j0 + k)];
  }
  __syncthreads();
  const int64_t c = (int64_t)j0 + jb + blockIdx.x * (int64_t)NT + threadIdx.x;
  if (c >= r) return;
  cplx x[kLuPanel];
  for (int i = 0; i < jb; ++i) {
    cplx v = W[(j0 + i) + n * c];
    for (int k = 0; k < i; ++k) {
      const cplx l = L[i + jb * k];
      v.x -= l.x * x[k].x - l.y * x[k].y;
      v.y -= l.x * x[k].y + l.y * x[k].x;
    }
    x[i] = v;
    W[(j0 + i) + n * c] = v;
  }
}

__global__ void __launch_bounds__(NT) k_lu_pivot(cplx* W, int64_t n, int r, int j, int* perm, const ArgMax* partials,
                                                 int nparts, int* bad) {
  __shared__ ArgMax sh[8];
  ArgMax best{-1.0, INT64_MAX, -1, j};
  for (int q = threadIdx.x; q < nparts; q += NT)
    if (better(partials[q].v, partials[q].key, best.v, best.key)) best = partials[q];
  block_argmax(best, sh);
  const int64_t p = best.i;
  if (best.v <= 0.0 || p < 0) {
    if (threadIdx.x == 0) *bad = 1;
    return;
  }
  if (p != j) {
    for (int c = threadIdx.x; c < r; c += NT) {
      const cplx t = W[j + n * c];
      W[j + n * c] = W[p + n * c];
      W[p + n * c] = t;
    }
    if (threadIdx.x == 0) {
      const int t = perm[j];
      perm[j] = perm[p];
      perm[p] = t;
    }
  }
}

__global__ void k_copy_lower(const cplx* W, int64_t n, int r, cplx* Lr) {
  const int64_t total = (int64_t)r * r;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
    const int64_t i = e / r, k = e % r;
    Lr[e] = k < i ? W[i + n * k] : cmk(0, 0);
  }
}

__global__ void __launch_bounds__(128) k_unit_lower_inverse(const cplx* Lr, int r, cplx* T) {
  extern __shared__ cplx tcol[];
  __shared__ double sh[8 * 2];
  const int c = blockIdx.x;
  for (int k = threadIdx.x; k < r; k += blockDim.x) tcol[k] = cmk(k == c ? 1.0 : 0.0, 0.0);
  __syncthreads();
  for (int i = c + 1; i < r; ++i) {
    double v[2] = {0, 0};
    const cplx* row = Lr + (int64_t)i * r;
    for (int k = c + threadIdx.x; k < i; k += blockDim.x) {
      const cplx l = row[k], t = tcol[k];
      v[0] += l.x * t.x - l.y * t.y;
      v[1] += l.x * t.y + l.y * t.x;
    }
    block_sum<2>(v, sh);
    if (threadIdx.x == 0) tcol[i] = cmk(-v[0], -v[1]);
    __syncthreads();
  }
  for (int k = threadIdx.x; k < r; k += blockDim.x) T[k + (int64_t)r * c] = tcol[k];
}

__global__ void k_set_identity_top(cplx* B, int64_t n, int r) {
  const int64_t total = (int64_t)r * r;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
    const int64_t i = e % r, c = e / r;
    B[i + n * c] = cmk(i == c ? 1.0 : 0.0, 0.0);
  }
}

__global__ void __launch_bounds__(NT) k_maxvol_update(cplx* B, int64_t n, int r, const int* perm, const cplx* rowbuf,
                                                      const MaxvolState* st, int update, ArgMax* partials) {
  extern __shared__ cplx rb[];
  __shared__ ArgMax sh[8];
  __shared__ int s_done, s_istar, s_cstar;
  __shared__ cplx s_inv;
  if (threadIdx.x == 0) {
    s_done = update ? st->done : 0;
    s_istar = st->i_star;
    s_cstar = st->c_star;
    const cplx pv = st->piv;
    const double d = cabs2(pv);
    s_inv = d > 0 ? cmk(pv.x / d, -pv.y / d) : cmk(0, 0);
  }
  __syncthreads();
  if (s_done) return;
  if (update)
    for (int c = threadIdx.x; c < r; c += NT) rb[c] = rowbuf[c];
  __syncthreads();
  const int cs = s_cstar;
  ArgMax best{-1.0, INT64_MAX, -1, 0};
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const int64_t key0 = (int64_t)perm[i] * r;
    if (update) {
      if (i == s_istar) {
        for (int c = 0; c < r; ++c) B[i + n * c] = cmk(c == cs ? 1.0 : 0.0, 0.0);
        if (better(1.0, key0 + cs, best.v, best.key)) { best.v = 1.0; best.key = key0 + cs; best.i = i; best.c = cs; }
        continue;
      }
      const cplx f = cmul(B[i + n * cs], s_inv);
      for (int c = 0; c < r; ++c) {
        const cplx u = rb[c];
        cplx w = B[i + n * c];
        w.x -= f.x * u.x - f.y * u.y;
        w.y -= f.x * u.y + f.y * u.x;
        B[i + n * c] = w;
        const double v = cabs2(w);
        if (better(v, key0 + c, best.v, best.key)) { best.v = v; best.key = key0 + c; best.i = i; best.c = c; }
      }
    } else {
      for (int c = 0; c < r; ++c) {
        const double v = cabs2(B[i + n * c]);
        if (better(v, key0 + c, best.v, best.key)) { best.v = v; best.key = key0 + c; best.i = i; best.c = c; }
      }
    }
  }
  block_argmax(best, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = best;
}

__global__ void __launch_bounds__(NT) k_maxvol_select(cplx* B, int64_t n, int r, const ArgMax* partials, int nparts,
                                                      double tau, int* piv_pos, cplx* rowbuf, MaxvolState* st) {
  __shared__ ArgMax sh[8];
  __shared__ int s_done;
  if (threadIdx.x == 0) s_done = st->done;
  __syncthreads();
  if (s_done) return;
  ArgMax best{-1.0, INT64_MAX, -1, 0};
  for (int q = threadIdx.x; q < nparts; q += NT)
    if (better(partials[q].v, partials[q].key, best.v, best.key)) best = partials[q];
  block_argmax(best, sh);
  const double m = sqrt(best.v);
  if (m <= 1.0 + tau || best.i < 0) {
    if (threadIdx.x == 0) {
      st->done = 1;
      st->maxabs = m;
    }
    return;
  }
  const int64_t i = best.i;
  const int c = best.c;
  for (int cc = threadIdx.x; cc < r; cc += NT) {
    cplx v = B[i + n * cc];
    if (cc == c) v.x -= 1.0;
    rowbuf[cc] = v;
  }
  if (threadIdx.x == 0) {
    st->i_star = (int)i;
    st->c_star = c;
    st->piv = B[i + n * c];
    st->maxabs = m;
    st->swaps += 1;
    piv_pos[c] = (int)i;
  }
}

__global__ void k_scatter_rows(const cplx* B, int64_t n, int r, const int* perm, cplx* Bout) {
  const int64_t total = n * r;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
    const int64_t i = e % n, c = e / n;
    Bout[perm[i] + n * c] = B[e];
  }
}

__global__ void k_add_diag(cplx* G, int q, double s) {
  for (int i = blockIdx.x * NT + threadIdx.x; i < q; i += gridDim.x * NT) G[i + (int64_t)q * i].x += s;
}

__global__ void k_trace_real(const cplx* G, int q, double* out) {
  double v[1] = {0};
  for (int i = threadIdx.x; i < q; i += NT) v[0] += G[i + (int64_t)q * i].x;
  __shared__ double sh[8];
  block_sum<1>(v, sh);
  if (threadIdx.x == 0) *out = v[0];
}

// one right-looking step j of the upper Cholesky on the unscaled rows:
// G[a, b] -= conj(G[j, a]) G[j, b] / G[j, j] for j < a <= b (upper part)
__global__ void k_chol_step(cplx* G, int q, int j) {
  const int64_t n = q - j - 1;
  const int64_t total = n * n;
  const double d = G[j + (int64_t)q * j].x;
  const double inv = d > 0 ? 1.0 / d : 0.0;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
    const int64_t a = j + 1 + e % n, b = j + 1 + e / n;
    if (a > b) continue;
    const cplx ga = G[j + (int64_t)q * a], gb = G[j + (int64_t)q * b];
    cplx v = G[a + (int64_t)q * b];
    // conj(ga) * gb * inv
    const double re = (ga.x * gb.x + ga.y * gb.y) * inv, im = (ga.x * gb.y - ga.y * gb.x) * inv;
    v.x -= re;
    v.y -= im;
    G[a + (int64_t)q * b] = v;
  }
}

// final scaling: R[j, c] = G[j, c] / sqrt(G[j, j]) (c > j), zero below the diagonal; the
// diagonal itself is written by k_chol_diag afterwards (scaling and overwriting it in one
// pass let some threads read an already replaced G[j, j]: a race that changed R run to run)
__global__ void k_chol_finish(cplx* G, int q, int* bad) {
  const int64_t total = (int64_t)q * q;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
    const int64_t j = e % q, c = e / q;
    if (j > c) {
      G[e] = cmk(0, 0);
      continue;
    }
    if (j == c) continue;
    const double d = G[j + (int64_t)q * j].x;
    if (!(d > 0)) {
      if (bad) *bad = 1;
      continue;
    }
    const double s = 1.0 / sqrt(d);
    const cplx v = G[e];
    G[e] = cmk(v.x * s, v.y * s);
  }
}

__global__ void k_chol_diag(cplx* G, int q, int* bad) {
  for (int j = blockIdx.x * NT + threadIdx.x; j < q; j += gridDim.x * NT) {
    const double d = G[j + (int64_t)q * j].x;
    if (!(d > 0)) {
      if (bad) *bad = 1;
      continue;
    }
    G[j + (int64_t)q * j] = cmk(sqrt(d), 0.0);
  }
}

// X[:, c] = R^{-1} e_c, back substitution on the row-major copy Rt (Rt[i q + k] = R[i, k])
__global__ void __launch_bounds__(128) k_upper_inverse(const cplx* Rt, int q, cplx* X) {
  extern __shared__ cplx xcol[];
  __shared__ double sh[8 * 2];
  const int c = blockIdx.x;
  for (int k = threadIdx.x; k < q; k += blockDim.x) xcol[k] = cmk(0, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    const cplx d = Rt[(int64_t)c * q + c];
    const double n2 = cabs2(d);
    xcol[c] = cmk(d.x / n2, -d.y / n2);
  }
  __syncthreads();
  for (int i = c - 1; i >= 0; --i) {
    double v[2] = {0, 0};
    const cplx* row = Rt + (int64_t)i * q;
    for (int k = i + 1 + threadIdx.x; k <= c; k += blockDim.x) {
      const cplx r = row[k], x = xcol[k];
      v[0] += r.x * x.x - r.y * x.y;
      v[1] += r.x * x.y + r.y * x.x;
    }
    block_sum<2>(v, sh);
    if (threadIdx.x == 0) {
      const cplx d = row[i];
      const double n2 = cabs2(d);
      const cplx di = cmk(d.x / n2, -d.y / n2);
      xcol[i] = cmul(cmk(-v[0], -v[1]), di);
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < q; k += blockDim.x) X[k + (int64_t)q * c] = xcol[k];
}

__global__ void k_gather_rows_owned(const cplx* src, int64_t lds, const int* idx, int nr, int64_t cols, int64_t r0,
                                    int64_t r1, cplx* dst) {
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < (int64_t)nr * cols; e += (int64_t)gridDim.x * NT) {
    const int i = (int)(e % nr);
    const int64_t c = e / nr;
    const int64_t row = idx[i];
    dst[e] = (row >= r0 && row < r1) ? src[(row - r0) + lds * c] : cmk(0, 0);
  }
}

__global__ void k_copy_conj(const cplx* src, int64_t lds, int64_t rows, int64_t cols, cplx* dst) {
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * NT) {
    const int64_t r = e % rows, c = e / rows;
    dst[e] = cconj(src[r + lds * c]);
  }
}

__global__ void k_conj_2d(cplx* C, int64_t ldc, int64_t rows, int64_t cols) {
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * NT) {
    const int64_t r = e % rows, c = e / rows;
    C[r + ldc * c].y = -C[r + ldc * c].y;
  }
}

unsigned grid1(int64_t work) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, NT), 148 * 16)); }

}  // namespace

void launch_gaussian(cplx* out, int64_t n, uint64_t seed, cudaStream_t st) {
  if (n <= 0) return;
  k_gaussian<<<grid1(n), NT, 0, st>>>(out, n, seed);
  VSIE_CHECK_LAUNCH();
}

void launch_jacobi_round(cplx* A, int64_t p, int64_t lda, cplx* V, int64_t q, const int2* pairs, int npairs,
                         double thr, double small2, unsigned* cnt, cudaStream_t st) {
  k_jacobi_round<<<npairs, NT, 0, st>>>(A, p, lda, V, q, pairs, thr, small2, cnt);
  VSIE_CHECK_LAUNCH();
}

bool launch_jacobi_coop(cplx* A, int64_t p, int64_t lda, cplx* V, int64_t q, const int2* pairs, int npairs,
                        int nrounds, double thr, double small2, int max_sweeps, unsigned* cnt, cudaStream_t st) {
  static int max_blocks = -1;
  if (max_blocks < 0) {
    int per_sm = 0, dev = 0, sms = 0;
    VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi_coop, NT, 0));
    VSIE_CHECK_CUDA(cudaGetDevice(&dev));
    VSIE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    max_blocks = per_sm * sms;
  }
  if (npairs > max_blocks) return false;
  void* args[] = {&A, &p, &lda, &V, &q, (void*)&pairs, &nrounds, &thr, &small2, &max_sweeps, &cnt};
  VSIE_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)k_jacobi_coop, dim3(npairs), dim3(NT), args, 0, st));
  VSIE_COUNT_LAUNCH();
  return true;
}

void launch_col_norms(const cplx* A, int64_t p, int64_t q, int64_t lda, double* out, cudaStream_t st) {
  if (q <= 0) return;
  k_col_norms<<<(unsigned)q, NT, 0, st>>>(A, p, lda, out);
  VSIE_CHECK_LAUNCH();
}

void launch_frob2(const cplx* A, int64_t n, double* partial, double* out, cudaStream_t st) {
  const int np = (int)std::min<int64_t>(1024, std::max<int64_t>(1, ceil_div(n, NT)));
  k_frob_partial<<<np, NT, 0, st>>>(A, n, partial);
  k_frob_final<<<1, 32, 0, st>>>(partial, np, out);
  VSIE_CHECK_LAUNCH();
}

void launch_gather_cols(const cplx* src, int64_t rows, int64_t lds, const int* idx, const double* scale, int ncols,
                        cplx* dst, int64_t ldd, bool conj, cudaStream_t st) {
  if (ncols <= 0 || rows <= 0) return;
  dim3 g((unsigned)std::min<int64_t>(ceil_div(rows, NT), 64), ncols);
  k_gather_cols<<<g, NT, 0, st>>>(src, rows, lds, idx, scale, ncols, dst, ldd, conj ? 1 : 0);
  VSIE_CHECK_LAUNCH();
}

void launch_gather_rows(const cplx* src, int64_t lds, const int* idx, int nr, int64_t cols, cplx* dst,
                        cudaStream_t st) {
  if (nr <= 0 || cols <= 0) return;
  k_gather_rows<<<grid1((int64_t)nr * cols), NT, 0, st>>>(src, lds, idx, nr, cols, dst);
  VSIE_CHECK_LAUNCH();
}

void launch_transpose(const cplx* src, int64_t R, int64_t C, cplx* dst, bool conj, cudaStream_t st) {
  if (R <= 0 || C <= 0) return;
  dim3 g((unsigned)ceil_div(R, 32), (unsigned)ceil_div(C, 32));
  k_transpose<<<g, NT, 0, st>>>(src, R, C, dst, conj ? 1 : 0);
  VSIE_CHECK_LAUNCH();
}

void launch_add_diag(cplx* G, int q, double s, cudaStream_t st) {
  k_add_diag<<<grid1(q), NT, 0, st>>>(G, q, s);
  VSIE_CHECK_LAUNCH();
}

void launch_trace_real(const cplx* G, int q, double* out, cudaStream_t st) {
  k_trace_real<<<1, NT, 0, st>>>(G, q, out);
  VSIE_CHECK_LAUNCH();
}

void launch_gather_rows_owned(const cplx* src, int64_t lds, const int* idx, int nr, int64_t cols, int64_t r0,
                              int64_t r1, cplx* dst, cudaStream_t st) {
  if (nr <= 0 || cols <= 0) return;
  k_gather_rows_owned<<<grid1((int64_t)nr * cols), NT, 0, st>>>(src, lds, idx, nr, cols, r0, r1, dst);
  VSIE_CHECK_LAUNCH();
}

void launch_copy_conj(const cplx* src, int64_t lds, int64_t rows, int64_t cols, cplx* dst, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  k_copy_conj<<<grid1(rows * cols), NT, 0, st>>>(src, lds, rows, cols, dst);
  VSIE_CHECK_LAUNCH();
}

void launch_conj_2d(cplx* C, int64_t ldc, int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  k_conj_2d<<<grid1(rows * cols), NT, 0, st>>>(C, ldc, rows, cols);
  VSIE_CHECK_LAUNCH();
}

void launch_cholesky_upper(cplx* G, int q, int* bad, cudaStream_t st) {
  for (int j = 0; j + 1 < q; ++j) {
    const int64_t n = q - j - 1;
    k_chol_step<<<grid1(n * n), NT, 0, st>>>(G, q, j);
    VSIE_CHECK_LAUNCH();
  }
  k_chol_finish<<<grid1((int64_t)q * q), NT, 0, st>>>(G, q, bad);
  VSIE_CHECK_LAUNCH();
  k_chol_diag<<<grid1(q), NT, 0, st>>>(G, q, bad);
  VSIE_CHECK_LAUNCH();
}

void launch_upper_inverse(const cplx* R, int q, cplx* Rt, cplx* X, cudaStream_t st) {
  launch_transpose(R, q, q, Rt, false, st);
  static bool configured = false;
  if (!configured) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_upper_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    configured = true;
  }
  k_upper_inverse<<<q, 128, (size_t)q * sizeof(cplx), st>>>(Rt, q, X);
  VSIE_CHECK_LAUNCH();
}

int lu_nparts(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, NT), 592)); }

void launch_lu_update(cplx* W, int64_t n, int r, int j, int c1, bool scale, bool argmax, ArgMax* partials, int nparts,
                      cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_lu_update, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_maxvol_update, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_unit_lower_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    configured = true;
  }
  k_lu_update<<<nparts, NT, (size_t)r * sizeof(cplx), st>>>(W, n, r, j, c1, scale ? 1 : 0, argmax ? 1 : 0, partials);
  VSIE_CHECK_LAUNCH();
}

void launch_lu_trsm(cplx* W, int64_t n, int r, int j0, int jb, cudaStream_t st) {
  if (j0 + jb >= r) return;
  k_lu_trsm<<<(unsigned)ceil_div(r - j0 - jb, NT), NT, 0, st>>>(W, n, r, j0, jb);
  VSIE_CHECK_LAUNCH();
}

void launch_lu_pivot(cplx* W, int64_t n, int r, int j, int* perm, const ArgMax* partials, int nparts, int* bad,
                     cudaStream_t st) {
  k_lu_pivot<<<1, NT, 0, st>>>(W, n, r, j, perm, partials, nparts, bad);
  VSIE_CHECK_LAUNCH();
}

void launch_copy_lower(const cplx* W, int64_t n, int r, cplx* Lr, cudaStream_t st) {
  k_copy_lower<<<grid1((int64_t)r * r), NT, 0, st>>>(W, n, r, Lr);
  VSIE_CHECK_LAUNCH();
}

void launch_unit_lower_inverse(const cplx* Lr, int r, cplx* T, cudaStream_t st) {
  k_unit_lower_inverse<<<r, 128, (size_t)r * sizeof(cplx), st>>>(Lr, r, T);
  VSIE_CHECK_LAUNCH();
}

void launch_set_identity_top(cplx* B, int64_t n, int r, cudaStream_t st) {
  k_set_identity_top<<<grid1((int64_t)r * r), NT, 0, st>>>(B, n, r);
  VSIE_CHECK_LAUNCH();
}

void launch_maxvol_update(cplx* B, int64_t n, int r, const int* perm, const cplx* rowbuf, const MaxvolState* s,
                          bool update, ArgMax* partials, int nparts, cudaStream_t st) {
  k_maxvol_update<<<nparts, NT, (size_t)r * sizeof(cplx), st>>>(B, n, r, perm, rowbuf, s, update ? 1 : 0, partials);
  VSIE_CHECK_LAUNCH();
}

void launch_maxvol_select(cplx* B, int64_t n, int r, const ArgMax* partials, int nparts, double tau, int* piv_pos,
                          cplx* rowbuf, MaxvolState* s, cudaStream_t st) {
  k_maxvol_select<<<1, NT, 0, st>>>(B, n, r, partials, nparts, tau, piv_pos, rowbuf, s);
  VSIE_CHECK_LAUNCH();
}

void launch_scatter_rows(const cplx* B, int64_t n, int r, const int* perm, cplx* Bout, cudaStream_t st) {
  k_scatter_rows<<<grid1(n * r), NT, 0, st>>>(B, n, r, perm, Bout);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
