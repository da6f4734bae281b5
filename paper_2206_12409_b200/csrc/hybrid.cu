// The GMRES consumer of the hybrid VSIE system (include/vsie_hybrid.h):
// the Eq. 15 operator composed from the library's block handles, and restarted GMRES with
// the Krylov basis, the projections and the updates on the device.
//
// Matvec: the input is staged into a fixed buffer X so that the coupling
// handles' captured CUDA graphs (keyed by pointers) are reused across GMRES iterations.
//   cb_far pair:  Y_b = Z_cb^f X_f, Y_f = (Z_cb^f)^T X_b      (one fused TT pair, apply.cu)
//   cb_near pair: T_b = Z_cb^n X_n, Y_n = (Z_cb^n)^T X_b
//   ff:           Y_f += Z_cc^ff X_f                          (farfar.cu, accumulate)
//   nn:           Y_n += Z_cc^nn X_n
//   fn pair:      T_n = U W^T X_f, T_f = W U^T X_n            (farnear.cu)
//   combine:      Y_f += T_f, Y_n += T_n, Y_b += T_b + d_b .* X_b   (one kernel)
// GMRES: oracle/gmres.py's order (CGS2 Arnoldi, Givens rotations, back substitution).  The
// projections h = V^H w are block partial sums over fixed row ranges reduced in block order,
// so every result is bitwise reproducible run to run.
#include "hybrid.hpp"

#include "farfar.hpp"
#include "farnear.hpp"
#include "handle.hpp"

#include <chrono>
#include <cmath>
#include <complex>
#include <vector>

struct vsie_hybrid_s {
  vsie_farfar_s* ff = nullptr;
  vsie_farnear_s* fn = nullptr;
  vsie_farfar_s* nn = nullptr;
  vsie_coupling_s* cbf = nullptr;
  vsie_coupling_s* cbn = nullptr;
  int64_t mf = 0, mn = 0, nb = 0, n = 0;
  int64_t matvecs = 0;
  vsie::DevBuf<vsie::cplx> d;       // [nb] body diagonal
  vsie::DevBuf<vsie::cplx> X, Y;    // [n] staged matvec input / output
  vsie::DevBuf<vsie::cplx> T;       // [mf + mn + nb] temporaries T_f | T_n | T_b
  vsie::DevBuf<vsie::cplx> V;       // [n x (restart + 1)] Krylov basis
  vsie::DevBuf<vsie::cplx> w, r;    // [n]
  vsie::DevBuf<vsie::cplx> part;    // projection partials [kBlocks x 128]
  vsie::DevBuf<double> npart;       // norm partials [kBlocks]
  vsie::DevBuf<vsie::cplx> hbuf;    // [restart + 1] coefficients on device
  vsie::DevBuf<double> nrm;         // [1]
};

namespace vsie {

namespace {

constexpr int kThreads = 256;
constexpr int kBlocks = 592;      // 4 per SM: fixed, so the partial-sum order never changes
constexpr int kChunk = 8;         // basis columns per projection pass

// partial[b * ldp + i] = sum over rows of block b of conj(V[r + ldv i]) w[r], i in [i0, i0 + kc)
__global__ void __launch_bounds__(kThreads) k_proj_partial(const cplx* __restrict__ V, int64_t ldv, int i0, int kc,
                                                           const cplx* __restrict__ w, int64_t n, cplx* partial,
                                                           int ldp) {
  __shared__ double sh[kThreads / 32][2 * kChunk];
  const int64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
  double acc[2 * kChunk];
#pragma unroll
  for (int q = 0; q < 2 * kChunk; ++q) acc[q] = 0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kThreads) {
    const cplx wv = w[r];
#pragma unroll
    for (int q = 0; q < kChunk; ++q)
      if (q < kc) {
        const cplx v = V[r + ldv * (i0 + q)];
        acc[2 * q] += v.x * wv.x + v.y * wv.y;       // Re(conj(v) w)
        acc[2 * q + 1] += v.x * wv.y - v.y * wv.x;   // Im(conj(v) w)
      }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 2 * kChunk; ++q)
    for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 2 * kChunk; ++q) sh[warp][q] = acc[q];
  __syncthreads();
  if (threadIdx.x < kc) {
    double re = 0, im = 0;
    for (int u = 0; u < kThreads / 32; ++u) {
      re += sh[u][2 * threadIdx.x];
      im += sh[u][2 * threadIdx.x + 1];
    }
    partial[(int64_t)blockIdx.x * ldp + i0 + threadIdx.x] = cmk(re, im);
  }
}

// h[i] = sum_b partial[b * ldp + i] (block order), i < k; one warp per i
__global__ void k_proj_reduce(const cplx* __restrict__ partial, int ldp, int nblk, int k, cplx* h) {
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= k) return;
  double re = 0, im = 0;
  for (int b = lane; b < nblk; b += 32) {
    const cplx p = partial[(int64_t)b * ldp + i];
    re += p.x;
    im += p.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) h[i] = cmk(re, im);
}

// w[r] += sgn sum_{i<k} V[r + ldv i] h[i]; npart[b] = sum over block b of |w[r]|^2 (new w)
__global__ void __launch_bounds__(kThreads) k_update(const cplx* __restrict__ V, int64_t ldv, int k,
                                                     const cplx* __restrict__ h, double sgn, cplx* w, int64_t n,
                                                     double* npart) {
  __shared__ cplx hs[128];
  __shared__ double sh[kThreads / 32];
  for (int i = threadIdx.x; i < k; i += kThreads) hs[i] = h[i];
  __syncthreads();
  const int64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
  double s = 0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kThreads) {
    cplx acc = cmk(0, 0);
    for (int i = 0; i < k; ++i) cfma(acc, V[r + ldv * i], hs[i]);
    cplx v = w[r];
    if (k > 0) {
      v.x += sgn * acc.x;
      v.y += sgn * acc.y;
      w[r] = v;
    }
    s += v.x * v.x + v.y * v.y;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int u = 0; u < kThreads / 32; ++u) t += sh[u];
    npart[blockIdx.x] = t;
  }
}

__global__ void k_norm_reduce(const double* npart, int nblk, double* out) {
  double s = 0;
  for (int b = threadIdx.x; b < nblk; b += 32) s += npart[b];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[0] = sqrt(s);
}

// out = a * in (real a)
__global__ void k_scale(const cplx* __restrict__ in, double a, cplx* out, int64_t n) {
  for (int64_t r = blockIdx.x * (int64_t)kThreads + threadIdx.x; r < n; r += (int64_t)gridDim.x * kThreads)
    out[r] = cmk(a * in[r].x, a * in[r].y);
}

// r = b - r
__global__ void k_rsub(const cplx* __restrict__ b, cplx* r, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    r[i] = csub(b[i], r[i]);
}

// Y_f += T_f, Y_n += T_n, Y_b += T_b (near domain only) and Y_b += d .* X_b (Y, T, X in the
// [f | n | b] layout)
__global__ void k_combine(cplx* Y, const cplx* __restrict__ T, const cplx* __restrict__ X, const cplx* __restrict__ d,
                          int64_t mfn, int64_t n, int has_near) {
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    cplx y = Y[i];
    if (has_near) y = cadd(y, T[i]);
    if (i >= mfn) cfma(y, d[i - mfn], X[i]);
    Y[i] = y;
  }
}

int grid_n(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kThreads), 148 * 16)); }

void hybrid_apply(vsie_hybrid_s* h, cudaStream_t st) {
  // Y = A X on the staged buffers
  cplx* X = h->X.p;
  cplx* Y = h->Y.p;
  cplx* T = h->T.p;
  const int64_t mf = h->mf, mn = h->mn;
  apply_pair(h->cbf, X, Y + mf + mn, X + mf + mn, Y, VSIE_OP_T, st);
  farfar_apply(h->ff, X, Y, VSIE_OP_N, 1, true, st);
  if (mn > 0) {
    apply_pair(h->cbn, X + mf, T + mf + mn, X + mf + mn, Y + mf, VSIE_OP_T, st);
    farfar_apply(h->nn, X + mf, Y + mf, VSIE_OP_N, 1, true, st);
    farnear_apply_pair(h->fn, X, T + mf, X + mf, T, st);
  }
  k_combine<<<grid_n(h->n), kThreads, 0, st>>>(Y, T, X, h->d.p, mf + mn, h->n, mn > 0 ? 1 : 0);
  VSIE_CHECK_LAUNCH();
  h->matvecs += 1;
}

// h[0..k) = V[:, 0..k)^H w (device), k <= restart + 1
void project(vsie_hybrid_s* h, const cplx* V, int64_t ldv, int k, const cplx* w, cplx* hout, cudaStream_t st) {
  const int ldp = 128;
  for (int i0 = 0; i0 < k; i0 += kChunk) {
    const int kc = std::min(kChunk, k - i0);
    k_proj_partial<<<kBlocks, kThreads, 0, st>>>(V, ldv, i0, kc, w, h->n, h->part.p, ldp);
    VSIE_CHECK_LAUNCH();
  }
  k_proj_reduce<<<(k + 7) / 8, 256, 0, st>>>(h->part.p, ldp, kBlocks, k, hout);
  VSIE_CHECK_LAUNCH();
}

// w += sgn V[:, 0..k) c; returns ||w|| (synchronous)
double update(vsie_hybrid_s* h, const cplx* V, int64_t ldv, int k, const cplx* c, double sgn, cplx* w,
              cudaStream_t st, bool want_norm) {
  k_update<<<kBlocks, kThreads, 0, st>>>(V, ldv, k, c, sgn, w, h->n, h->npart.p);
  VSIE_CHECK_LAUNCH();
  if (!want_norm) return 0;
  k_norm_reduce<<<1, 32, 0, st>>>(h->npart.p, kBlocks, h->nrm.p);
  VSIE_CHECK_LAUNCH();
  double v = 0;
  VSIE_CHECK_CUDA(cudaMemcpyAsync(&v, h->nrm.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
  return v;
}

double norm(vsie_hybrid_s* h, const cplx* v, cudaStream_t st) {
  // ||v|| through the update kernel with k = 0 (w unchanged, norm partials)
  return update(h, nullptr, 0, 0, h->hbuf.p, 0.0, const_cast<cplx*>(v), st, true);
}

}  // namespace

vsie_hybrid_s* hybrid_new() { return new vsie_hybrid_s(); }
void hybrid_delete(vsie_hybrid_s* h) { delete h; }

void hybrid_info(vsie_hybrid_s* h, vsie_hybrid_info* out) {
  out->m_far = h->mf;
  out->m_near = h->mn;
  out->n_body = h->nb;
  out->n = h->n;
  out->matvecs = h->matvecs;
}

void hybrid_create(vsie_farfar_s* ff, vsie_farnear_s* fn, vsie_farfar_s* nn, vsie_coupling_s* cbf,
                   vsie_coupling_s* cbn, const void* d_body, vsie_hybrid_s* h) {
  VSIE_REQUIRE(ff && cbf && d_body, VSIE_ERR_ARG, "hybrid: ff, cb_far and d_body are required");
  const bool near = fn || nn || cbn;
  VSIE_REQUIRE(!near || (fn && nn && cbn), VSIE_ERR_ARG, "hybrid: fn, nn and cb_near must be all set or all NULL");
  VSIE_REQUIRE(cbf->has_cores && cbf->world == 1, VSIE_ERR_ARG, "hybrid: cb_far must be a built single-process handle");
  VSIE_REQUIRE(ff->m == cbf->m, VSIE_ERR_ARG, "hybrid: Z_cc^ff and Z_cb^f disagree on m_f");
  h->ff = ff;
  h->cbf = cbf;
  h->mf = ff->m;
  h->nb = 3 * cbf->grid.nv();
  if (near) {
    VSIE_REQUIRE(cbn->has_cores && cbn->world == 1, VSIE_ERR_ARG, "hybrid: cb_near must be a built single-process handle");
    VSIE_REQUIRE(fn->mf == ff->m, VSIE_ERR_ARG, "hybrid: U V^* columns != m_f");
    VSIE_REQUIRE(fn->mn == nn->m && nn->m == cbn->m, VSIE_ERR_ARG, "hybrid: Z_cc^fn rows, Z_cc^nn and Z_cb^n disagree on m_n");
    for (int a = 0; a < 3; ++a)
      VSIE_REQUIRE(cbn->grid.n[a] == cbf->grid.n[a], VSIE_ERR_ARG, "hybrid: cb_near and cb_far on different grids");
    h->fn = fn;
    h->nn = nn;
    h->cbn = cbn;
    h->mn = nn->m;
  }
  h->n = h->mf + h->mn + h->nb;
  h->d.alloc(h->nb);
  VSIE_CHECK_CUDA(cudaMemcpy(h->d.p, d_body, h->nb * sizeof(cplx), cudaMemcpyDeviceToDevice));
  h->X.alloc(h->n);
  h->Y.alloc(h->n);
  h->T.alloc(h->n);
  h->part.alloc((size_t)kBlocks * 128);
  h->npart.alloc(kBlocks);
  h->nrm.alloc(1);
  h->hbuf.alloc(128);
}

void hybrid_matvec(vsie_hybrid_s* h, const void* x, void* y, cudaStream_t st) {
  VSIE_REQUIRE(x && y && x != y, VSIE_ERR_ARG, "hybrid_matvec: x / y NULL or aliased");
  VSIE_CHECK_CUDA(cudaMemcpyAsync(h->X.p, x, h->n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
  hybrid_apply(h, st);
  VSIE_CHECK_CUDA(cudaMemcpyAsync(y, h->Y.p, h->n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
}

int hybrid_gmres(vsie_hybrid_s* h, const void* bv, void* xv, int restart, int max_iter, double tol, double* history,
                 vsie_gmres_info* info, cudaStream_t st) {
  VSIE_REQUIRE(bv && xv && bv != xv, VSIE_ERR_ARG, "gmres: b / x NULL or aliased");
  VSIE_REQUIRE(restart >= 1 && restart <= 127 && max_iter >= 1 && tol > 0 && std::isfinite(tol), VSIE_ERR_ARG,
               "gmres: restart in 1..127, max_iter >= 1, tol > 0");
  using C = std::complex<double>;
  const auto t0 = std::chrono::steady_clock::now();
  const cplx* b = static_cast<const cplx*>(bv);
  cplx* x = static_cast<cplx*>(xv);
  const int64_t n = h->n, m = restart;
  h->V.ensure(n * (m + 1));
  h->w.ensure(n);
  h->r.ensure(n);
  cplx* V = h->V.p;
  cudaEvent_t e0, e1;
  VSIE_CHECK_CUDA(cudaEventCreate(&e0));
  VSIE_CHECK_CUDA(cudaEventCreate(&e1));
  double mv_ms = 0;
  auto matvec_into = [&](const cplx* in, cplx* out) {
    VSIE_CHECK_CUDA(cudaMemcpyAsync(h->X.p, in, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    VSIE_CHECK_CUDA(cudaEventRecord(e0, st));
    hybrid_apply(h, st);
    VSIE_CHECK_CUDA(cudaEventRecord(e1, st));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(out, h->Y.p, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    VSIE_CHECK_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    VSIE_CHECK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    mv_ms += ms;
  };
  VSIE_CHECK_CUDA(cudaMemsetAsync(x, 0, n * sizeof(cplx), st));
  const double bn = norm(h, b, st);
  int its = 0, cycles = 0;
  double rel = 0;
  if (bn > 0) {
    rel = 1.0;
    std::vector<C> H((size_t)(m + 1) * m), g(m + 1), hv(m + 1), h2(m + 1), sn(m), y(m);
    std::vector<double> cs(m);
    while (its < max_iter) {
      cplx* r = h->r.p;
      if (its == 0) {
        VSIE_CHECK_CUDA(cudaMemcpyAsync(r, b, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      } else {
        matvec_into(x, r);
        k_rsub<<<grid_n(n), kThreads, 0, st>>>(b, r, n);
        VSIE_CHECK_LAUNCH();
      }
      const double beta = norm(h, r, st);
      rel = beta / bn;
      if (rel <= tol) break;
      std::fill(H.begin(), H.end(), C(0));
      std::fill(g.begin(), g.end(), C(0));
      g[0] = beta;
      k_scale<<<grid_n(n), kThreads, 0, st>>>(r, 1.0 / beta, V, n);
      VSIE_CHECK_LAUNCH();
      int j = 0;
      while (j < m && its < max_iter) {
        cplx* w = h->w.p;
        matvec_into(V + n * j, w);
        ++its;
        // CGS2: h = V^H w, w -= V h; h2 = V^H w, w -= V h2 (norm of the result); h += h2
        project(h, V, n, j + 1, w, h->hbuf.p, st);
        update(h, V, n, j + 1, h->hbuf.p, -1.0, w, st, false);
        VSIE_CHECK_CUDA(cudaMemcpyAsync(hv.data(), h->hbuf.p, (j + 1) * sizeof(cplx), cudaMemcpyDeviceToHost, st));
        project(h, V, n, j + 1, w, h->hbuf.p, st);
        const double hn = update(h, V, n, j + 1, h->hbuf.p, -1.0, w, st, true);
        VSIE_CHECK_CUDA(cudaMemcpy(h2.data(), h->hbuf.p, (j + 1) * sizeof(cplx), cudaMemcpyDeviceToHost));
        C* col = &H[(size_t)j * (m + 1)];
        for (int i = 0; i <= j; ++i) col[i] = hv[i] + h2[i];
        col[j + 1] = hn;
        if (hn > 0) {
          k_scale<<<grid_n(n), kThreads, 0, st>>>(w, 1.0 / hn, V + n * (j + 1), n);
          VSIE_CHECK_LAUNCH();
        }
        // Givens rotations on the new column (oracle/gmres.py)
        for (int i = 0; i < j; ++i) {
          const C t = cs[i] * col[i] + sn[i] * col[i + 1];
          col[i + 1] = -std::conj(sn[i]) * col[i] + cs[i] * col[i + 1];
          col[i] = t;
        }
        double c;
        C s;
        const C a = col[j], bb = col[j + 1];
        if (bb == C(0)) {
          c = 1.0;
          s = 0.0;
        } else if (a == C(0)) {
          c = 0.0;
          s = std::conj(bb) / std::abs(bb);
        } else {
          const double t = std::hypot(std::abs(a), std::abs(bb));
          c = std::abs(a) / t;
          s = (a / std::abs(a)) * std::conj(bb) / t;
        }
        cs[j] = c;
        sn[j] = s;
        col[j] = c * col[j] + s * col[j + 1];
        col[j + 1] = 0;
        g[j + 1] = -std::conj(s) * g[j];
        g[j] = c * g[j];
        ++j;
        rel = std::abs(g[j]) / bn;
        if (history) history[its - 1] = rel;
        if (rel <= tol || hn == 0) break;
      }
      // y = R^{-1} g (back substitution), x += V y
      for (int i = j - 1; i >= 0; --i) {
        C acc = g[i];
        for (int k = i + 1; k < j; ++k) acc -= H[(size_t)k * (m + 1) + i] * y[k];
        y[i] = acc / H[(size_t)i * (m + 1) + i];
      }
      VSIE_CHECK_CUDA(cudaMemcpyAsync(h->hbuf.p, y.data(), j * sizeof(cplx), cudaMemcpyHostToDevice, st));
      update(h, V, n, j, h->hbuf.p, 1.0, x, st, false);
      VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
      ++cycles;
      if (rel <= tol) break;
    }
  }
  VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (info) {
    info->iterations = its;
    info->restarts = cycles;
    info->converged = rel <= tol ? 1 : 0;
    info->rel_residual = rel;
    info->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    info->matvec_seconds = mv_ms * 1e-3;
  }
  return rel <= tol ? VSIE_OK : VSIE_WARN_NOT_CONVERGED;
}

}  // namespace vsie
