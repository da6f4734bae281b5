// Blocked Householder QR of a tall complex matrix (the rank-revealing factorisations of the
// TT-cross driver: QR of the range-finder sketch and of the projected
// supercore, then a Jacobi SVD of the small R factor only).
//
// A (p x q, p >= q, column-major, ld lda) = Q R, Q = H_0 H_1 ... H_{q-1}, H_j = I - tau_j v_j v_j^H
// (LAPACK zgeqrf conventions: v_j[j] = 1, v_j[i < j] = 0; on exit R is in the upper triangle
// and v_j below the diagonal).  Backward stable for any condition number and rank (no Gram
// matrix, so singular values down to u ||A|| survive -- the cross's truncation sits near
// 1e-8 of the largest singular value at cfg 3).
//   * panels of up to kPB = 32 columns (narrower for very tall factors, so that a panel stays
//     in L2 across its column steps), each factorised by ONE cooperative launch: every CTA owns a
//     row range; per column two grid barriers (the norm, then the dot products with the
//     remaining panel columns), partial sums written per CTA and summed in fixed CTA order by
//     every CTA (deterministic);
//   * the compact WY form Q_panel = I - V T V^H (T upper triangular, LAPACK zlarft, from the
//     Gram matrix V^H V) and the trailing update A_t -= V (T^H (V^H A_t)) by three ZGEMMs;
//   * Q (or Q C) is applied panel by panel in reverse order by the same three ZGEMMs.
#include "crosskern.cuh"
#include "kernels.cuh"

#include <cooperative_groups.h>

#include <algorithm>

namespace vsie {
namespace {

constexpr int HT = 256;
constexpr int kPB = 32;                  // maximum panel width (T factors are stored kPB x kPB)
constexpr int kPS = 2 * kPB + 2;         // doubles per CTA partial record

// sum of N doubles over the CTA (result valid in every thread)
template <int N>
__device__ __forceinline__ void cta_sum(double (&v)[N], double* sh /* >= 8 N */) {
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
    for (int q = 0; q < HT / 32; ++q) s += sh[q * N + k];
    v[k] = s;
  }
  __syncthreads();
}

template <int PB>
__global__ void __launch_bounds__(HT) k_hqr_panel(cplx* A, int64_t lda, int64_t p, int j0, int jb, cplx* tau,
                                                  double* part) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[8 * 2 * PB];
  __shared__ double bc[5];   // beta, tau re / im, scale re / im broadcast
  __shared__ cplx wsh[PB];
  const int G = gridDim.x, blk = blockIdx.x;
  const int64_t L = p - j0;
  const int64_t r0 = j0 + L * blk / G, r1 = j0 + L * (blk + 1) / G;   // my rows
  for (int jj = 0; jj < jb; ++jj) {
    const int64_t j = j0 + jj;
    cplx* x = A + lda * j;
    // a. partial |x|^2 over my rows below the diagonal
    {
      double v[1] = {0};
      for (int64_t r = std::max(r0, j + 1) + threadIdx.x; r < r1; r += HT) v[0] += cabs2(x[r]);
      cta_sum<1>(v, sh);
      if (threadIdx.x == 0) part[(int64_t)blk * kPS] = v[0];
    }
    grid.sync();
    // c. the reflector (every CTA computes it from the same partials, fixed order)
    if (threadIdx.x == 0) {
      double xn2 = 0;
      for (int b = 0; b < G; ++b) xn2 += part[(int64_t)b * kPS];
      const cplx alpha = x[j];
      double tr = 0, ti = 0, sr = 0, si = 0, beta = alpha.x;
      if (!(xn2 == 0 && alpha.y == 0)) {
        const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn2);
        beta = alpha.x >= 0 ? -nrm : nrm;
        tr = (beta - alpha.x) / beta;
        ti = -alpha.y / beta;
        // scale = 1 / (alpha - beta)
        const double dr = alpha.x - beta, di = alpha.y, dn = dr * dr + di * di;
        sr = dr / dn;
        si = -di / dn;
      }
      bc[0] = beta;
      bc[1] = tr;
      bc[2] = ti;
      bc[3] = sr;
      bc[4] = si;
    }
    __syncthreads();
    const double beta = bc[0];
    const cplx t = cmk(bc[1], bc[2]), scl = cmk(bc[3], bc[4]);
    const bool active = !(t.x == 0 && t.y == 0);
    __syncthreads();
    if (active)
      for (int64_t r = std::max(r0, j + 1) + threadIdx.x; r < r1; r += HT) x[r] = cmul(x[r], scl);
    __syncthreads();
    // d. partial w_c = v^H A[:, c] over my rows (v[j] = 1), c = jj + 1 .. jb - 1
    const int nc = jb - jj - 1;
    if (active && nc > 0) {
      double v[2 * PB];
#pragma unroll
      for (int c = 0; c < 2 * PB; ++c) v[c] = 0;
      for (int64_t r = std::max(r0, j) + threadIdx.x; r < r1; r += HT) {
        const cplx vr = r == j ? cmk(1, 0) : x[r];
#pragma unroll
        for (int c = 0; c < PB; ++c)
          if (c < nc) {
            const cplx a = A[r + lda * (j + 1 + c)];
            v[2 * c] += vr.x * a.x + vr.y * a.y;       // conj(v) a
            v[2 * c + 1] += vr.x * a.y - vr.y * a.x;
          }
      }
      cta_sum<2 * PB>(v, sh);
      if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < 2 * PB; ++c)
          if (c < 2 * nc) part[(int64_t)blk * kPS + 2 + c] = v[c];
    }
    grid.sync();
    // f. A[:, c] -= conj(tau) v w_c on my rows; the diagonal becomes beta
    if (active && nc > 0) {
      if (threadIdx.x < nc) {
        double wr = 0, wi = 0;
        for (int b = 0; b < G; ++b) {
          wr += part[(int64_t)b * kPS + 2 + 2 * threadIdx.x];
          wi += part[(int64_t)b * kPS + 3 + 2 * threadIdx.x];
        }
        // conj(tau) w
        wsh[threadIdx.x] = cmk(t.x * wr + t.y * wi, t.x * wi - t.y * wr);
      }
      __syncthreads();
      for (int64_t r = std::max(r0, j) + threadIdx.x; r < r1; r += HT) {
        const cplx vr = r == j ? cmk(1, 0) : x[r];
        for (int c = 0; c < nc; ++c) {
          cplx& a = A[r + lda * (j + 1 + c)];
          a = csub(a, cmul(vr, wsh[c]));
        }
      }
    }
    if (r0 <= j && j < r1 && threadIdx.x == 0) {
      x[j] = cmk(beta, 0);
      tau[j] = t;
    }
    __syncthreads();
  }
}

// V (L x jb, ld L) of the panel: unit lower trapezoidal from the reflectors below the diagonal
__global__ void k_hqr_extract_v(const cplx* A, int64_t lda, int64_t p, int j0, int jb, cplx* V) {
  const int64_t L = p - j0;
  for (int64_t e = blockIdx.x * (int64_t)HT + threadIdx.x; e < L * jb; e += (int64_t)gridDim.x * HT) {
    const int64_t r = e % L;
    const int a = (int)(e / L);
    V[e] = r < a ? cmk(0, 0) : (r == a ? cmk(1, 0) : A[j0 + r + lda * (j0 + a)]);
  }
}

// T (jb x jb upper, ld kPB) of Q_panel = I - V T V^H from Gv = V^H V and tau (zlarft, forward
// columnwise): T[i][i] = tau_i, T[0:i, i] = -tau_i T[0:i, 0:i] Gv[0:i, i]
__global__ void k_hqr_t(const cplx* Gv, int jb, const cplx* tau, cplx* T) {
  __shared__ cplx Ts[kPB * kPB];
  for (int e = threadIdx.x; e < kPB * kPB; e += blockDim.x) Ts[e] = cmk(0, 0);
  __syncthreads();
  for (int i = 0; i < jb; ++i) {
    const cplx ti = tau[i];
    cplx s = cmk(0, 0);
    const int k = threadIdx.x;
    if (k < i)
      for (int l = k; l < i; ++l) s = cadd(s, cmul(Ts[k + kPB * l], Gv[l + jb * i]));
    __syncthreads();
    if (k < i) Ts[k + kPB * i] = cmul(cmk(-ti.x, -ti.y), s);
    if (k == i) Ts[i + kPB * i] = ti;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kPB * kPB; e += blockDim.x) T[e] = Ts[e];
}

// C[0:q, :] = B (q x n, ld ldb), C[q:p, :] = 0
__global__ void k_hqr_pad(const cplx* B, int64_t ldb, int q, int64_t p, int n, cplx* C, int64_t ldc, int identity) {
  for (int64_t e = blockIdx.x * (int64_t)HT + threadIdx.x; e < p * n; e += (int64_t)gridDim.x * HT) {
    const int64_t r = e % p;
    const int c = (int)(e / p);
    cplx v = cmk(0, 0);
    if (identity)
      v = r == c ? cmk(1, 0) : cmk(0, 0);
    else if (r < q)
      v = B[r + ldb * c];
    C[r + ldc * c] = v;
  }
}

// R (q x q) = the upper triangle of A, zero below
__global__ void k_hqr_r(const cplx* A, int64_t lda, int q, cplx* R) {
  for (int64_t e = blockIdx.x * (int64_t)HT + threadIdx.x; e < (int64_t)q * q; e += (int64_t)gridDim.x * HT) {
    const int64_t r = e % q, c = e / q;
    R[e] = r <= c ? A[r + lda * c] : cmk(0, 0);
  }
}

void gemm(Trans ta, Trans tb, int64_t M, int64_t N, int64_t K, cplx alpha, const cplx* A, int64_t lda, const cplx* B,
          int64_t ldb, cplx beta, cplx* C, int64_t ldc, const HqrWs& w, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  Zgemm z{};
  z.nbatch = 1;
  z.ta = ta;
  z.tb = tb;
  z.M[0] = M; z.N[0] = N; z.K[0] = K;
  z.A[0] = A; z.lda[0] = lda;
  z.B[0] = B; z.ldb[0] = ldb;
  z.C[0] = C; z.ldc[0] = ldc;
  z.alpha = alpha;
  z.beta = beta;
  launch_zgemm(z, w.zws, w.zws_elems, st);
}

unsigned grid1h(int64_t work) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, HT), 148 * 16)); }

int coop_ctas() {
  static int n = -1;
  if (n < 0) {
    int per_sm = 0, dev = 0, sms = 0;
    VSIE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hqr_panel<kPB>, HT, 0));
    VSIE_CHECK_CUDA(cudaGetDevice(&dev));
    VSIE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    n = std::max(1, std::min(per_sm, 2) * sms);
  }
  return n;
}

}  // namespace

int hqr_panels(int q) { return (q + 7) / 8; }   // upper bound on the panel count (width >= 8): T storage
int hqr_panel_width() { return kPB; }

// panel width for a factorisation of p rows: the panel (p x width complex) should stay in L2
// across its column steps (<= 48 MB), so very tall factors take narrower panels
int panel_width(int64_t p) {
  int b = kPB;
  while (b > 8 && (int64_t)p * b * 16 > (48LL << 20)) b /= 2;
  return b;
}

void hqr_factor(cplx* A, int64_t lda, int64_t p, int q, cplx* tau, cplx* T, const HqrWs& w, cudaStream_t st) {
  VSIE_REQUIRE(p >= q && q >= 1, VSIE_ERR_ARG, "hqr: need p >= q >= 1");
  const int bw = panel_width(p);
  for (int j0 = 0; j0 < q; j0 += bw) {
    const int jb = std::min(bw, q - j0);
    const int64_t L = p - j0;
    // cooperative panel factorisation: >= 64 rows per CTA
    int G = (int)std::max<int64_t>(1, std::min<int64_t>(coop_ctas(), L / 64));
    int j0a = j0, jba = jb;
    int64_t ldaa = lda, pa = p;
    double* part = w.part;
    cplx* taub = tau;   // indexed by the global column inside the kernel
    void* args[] = {&A, &ldaa, &pa, &j0a, &jba, &taub, &part};
    const void* fn = bw == 32 ? (const void*)k_hqr_panel<32> : bw == 16 ? (const void*)k_hqr_panel<16> : (const void*)k_hqr_panel<8>;
    VSIE_CHECK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(HT), args, 0, st));
    VSIE_COUNT_LAUNCH();
    // compact WY factor of the panel
    cplx* V = w.V;
    k_hqr_extract_v<<<grid1h(L * jb), HT, 0, st>>>(A, lda, p, j0, jb, V);
    VSIE_CHECK_LAUNCH();
    gemm(kC, kN, jb, jb, L, cmk(1, 0), V, L, V, L, cmk(0, 0), w.Gv, jb, w, st);
    cplx* Tp = T + (int64_t)(j0 / bw) * kPB * kPB;
    k_hqr_t<<<1, 32, 0, st>>>(w.Gv, jb, tau + j0, Tp);
    VSIE_CHECK_LAUNCH();
    // trailing update A_t -= V (T^H (V^H A_t))
    const int n = q - j0 - jb;
    if (n > 0) {
      cplx* At = A + j0 + lda * (j0 + jb);
      gemm(kC, kN, jb, n, L, cmk(1, 0), V, L, At, lda, cmk(0, 0), w.W, jb, w, st);
      gemm(kC, kN, jb, n, jb, cmk(1, 0), Tp, kPB, w.W, jb, cmk(0, 0), w.W2, jb, w, st);
      gemm(kN, kN, L, n, jb, cmk(-1, 0), V, L, w.W2, jb, cmk(1, 0), At, lda, w, st);
    }
  }
}

void hqr_apply_q(const cplx* A, int64_t lda, int64_t p, int q, const cplx* T, cplx* C, int64_t ldc, int n,
                 const HqrWs& w, cudaStream_t st) {
  const int bw = panel_width(p);
  const int np = (q + bw - 1) / bw;
  for (int pi = np - 1; pi >= 0; --pi) {
    const int j0 = pi * bw, jb = std::min(bw, q - j0);
    const int64_t L = p - j0;
    k_hqr_extract_v<<<grid1h(L * jb), HT, 0, st>>>(A, lda, p, j0, jb, w.V);
    VSIE_CHECK_LAUNCH();
    cplx* Cs = C + j0;
    const cplx* Tp = T + (int64_t)pi * kPB * kPB;
    gemm(kC, kN, jb, n, L, cmk(1, 0), w.V, L, Cs, ldc, cmk(0, 0), w.W, jb, w, st);
    gemm(kN, kN, jb, n, jb, cmk(1, 0), Tp, kPB, w.W, jb, cmk(0, 0), w.W2, jb, w, st);
    gemm(kN, kN, L, n, jb, cmk(-1, 0), w.V, L, w.W2, jb, cmk(1, 0), Cs, ldc, w, st);
  }
}

void hqr_fill(const cplx* B, int64_t ldb, int q, int64_t p, int n, cplx* C, int64_t ldc, bool identity,
              cudaStream_t st) {
  k_hqr_pad<<<grid1h(p * n), HT, 0, st>>>(B, ldb, q, p, n, C, ldc, identity ? 1 : 0);
  VSIE_CHECK_LAUNCH();
}

void hqr_copy_r(const cplx* A, int64_t lda, int q, cplx* R, cudaStream_t st) {
  k_hqr_r<<<grid1h((int64_t)q * q), HT, 0, st>>>(A, lda, q, R);
  VSIE_CHECK_LAUNCH();
}

size_t hqr_part_doubles() { return (size_t)coop_ctas() * kPS; }

}  // namespace vsie
