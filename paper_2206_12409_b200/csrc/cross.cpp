// DMRG two-site TT-cross of Z_bc, per chi (PAPER.md P:126-128, P:174-182,
// Eq. 14; readings R1-R3).
//
// Host C++ orchestration of device kernels:
//   for chi in {x, y, z}: r = (1, 1, 1), right index sets from one seeded index;
//   sweep: L->R k = 1..3, R->L k = 3..1:
//     M_k  = A(I_{<=k-1}, i_k, i_{k+1}, J_{>k+1})        entry kernel (block mode)
//     rank-revealing factorisation of M_k                  one-sided Jacobi SVD, directly
//                                                          or on randomized sketches
//     pivots + interpolation matrix                        maxvol (LU init, rank-1 updates)
//     cores: L->R  core_k = L L[P]^{-1}, G4 = M_3[P, :]
//            R->L  core_{k+1} = (R R[Q]^{-1})^T, G1 = M_1[:, Q]
//   stop when the ranks are unchanged over a sweep and the held-out error <= 10 tol.
// Multi-process (NCCL or the single-GPU IPC transport): supercore ROWS are split across the
// ranks: each rank evaluates and keeps its row block; the randomized range
// finder's products and sums run on the blocks (allgather of the sketch rows / allreduce of
// Q^H M), small factorisations are replicated (deterministic).
#include "cross.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <map>
#include <numeric>
#include <set>
#include <string>

#include "crosskern.cuh"
#include "kernels.cuh"

namespace vsie {

namespace {

using Clock = std::chrono::steady_clock;

uint64_t host_splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Ws {
  DevBuf<cplx> M, J, V, Y, Q, Bh, basis, Bp, Bout, T, Lr, omega, Vr, rowbuf;
  DevBuf<cplx> G, Rinv, Rt, Rtmp, Ra, Rb, Atmp, zws, other;
  DevBuf<cplx> tau, Th, Vh, W, W2, Gv;   // blocked Householder QR (hqr.cu)
  DevBuf<cplx> Bc, Yraw;                 // conj(B) staging of zgemm_tc; raw sketch M Omega
  DevBuf<cplx> gsend, grecv, Mfull, Yloc, Bloc;   // row-split build: allgather staging, assembled blocks
  DevBuf<double> hpart;
  DevBuf<double> norms, frob_partial, frob;
  DevBuf<int> perm, piv_pos, idx, bad;
  DevBuf<ArgMax> partials;
  DevBuf<MaxvolState> mvs;
  DevBuf<unsigned> rotcnt;
  DevBuf<int32_t> left, right;
  std::map<int, DevBuf<int2>> schedules;
};

struct Ctx {
  vsie_coupling_s* h;
  vsie_build_opts o;
  cudaStream_t st;
  Ws ws;
  double tol, delta;
  uint64_t seed;
  uint64_t sketch_counter = 0;
  double t_entry = 0, t_factor = 0, t_maxvol = 0, t_maxvol_lu = 0;
  int64_t maxvol_swaps = 0;
  int64_t n_eval = 0;
  int64_t jacobi_sweeps = 0;
  double t_jsmall = 0, t_chol = 0, t_gemm = 0;
  // multi-process build (SURVEY §8e cross step): the supercore's ROWS are split over the
  // ranks; this rank holds rows [rp0, rp1) of the current M (ld rp1 - rp0)
  bool dist = false;
  int64_t rp0 = 0, rp1 = 0;
};

void sync(Ctx& c) { VSIE_CHECK_CUDA(cudaStreamSynchronize(c.st)); }

double secs(Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); }

// ------------------------------------------------------------------ one-sided Jacobi
const int2* schedule(Ctx& c, int Q) {
  auto it = c.ws.schedules.find(Q);
  if (it != c.ws.schedules.end()) return it->second.p;
  std::vector<int2> pairs;
  pairs.reserve((size_t)(Q - 1) * (Q / 2));
  std::vector<int> L(Q);
  for (int t = 0; t < Q - 1; ++t) {
    L[0] = 0;
    for (int i = 0; i < Q - 1; ++i) L[i + 1] = (t + i) % (Q - 1) + 1;
    for (int k = 0; k < Q / 2; ++k) pairs.push_back(make_int2(L[k], L[Q - 1 - k]));
  }
  DevBuf<int2>& d = c.ws.schedules[Q];
  d.alloc(pairs.size());
  VSIE_CHECK_CUDA(cudaMemcpy(d.p, pairs.data(), pairs.size() * sizeof(int2), cudaMemcpyHostToDevice));
  return d.p;
}

// Orthogonalises the columns of A (p x q, ld p); accumulates rotations into V (q x q) if given.
// small_rel: columns with norm below small_rel ||A||_F are left unrotated (numerical zeros
// for 1e-14; for the truncated factorisations of the cross, columns 100x below the
// truncation level delta can neither be kept nor move the kept singular values)
void jacobi(Ctx& c, cplx* A, int64_t p, int q, cplx* V, double small_rel = 1e-14) {
  if (q <= 1) return;
  const int Q = q + (q & 1);
  const int2* sch = schedule(c, Q);
  c.ws.rotcnt.ensure(1);
  // rotation threshold on |a_i^H a_j| / (|a_i| |a_j|): 1e-12.  One-sided Jacobi
  // keeps relative accuracy per singular value, so a residual cosine of 1e-12
  // perturbs each sigma by ~1e-12 relative — far below the truncation levels
  // (tol / sqrt 3 >= 5.8e-9) — while avoiding the long tail of sweeps that
  // a sqrt(p) eps threshold spends on rounding noise.
  const double thr = std::max(1e-12, std::sqrt((double)p) * 2.3e-16);
  c.ws.frob_partial.ensure(1024);
  c.ws.frob.ensure(1);
  launch_frob2(A, p * q, c.ws.frob_partial.p, c.ws.frob.p, c.st);
  double fro2 = 0;
  VSIE_CHECK_CUDA(cudaMemcpyAsync(&fro2, c.ws.frob.p, sizeof(double), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  const double small2 = small_rel * small_rel * fro2;
  c.ws.rotcnt.ensure(3);
  VSIE_CHECK_CUDA(cudaMemsetAsync(c.ws.rotcnt.p, 0, 3 * sizeof(unsigned), c.st));
  if (launch_jacobi_coop(A, p, p, V, q, sch, Q / 2, Q - 1, thr, small2, 40, c.ws.rotcnt.p, c.st)) {
    unsigned hs[3];
    VSIE_CHECK_CUDA(cudaMemcpyAsync(hs, c.ws.rotcnt.p, sizeof(hs), cudaMemcpyDeviceToHost, c.st));
    sync(c);
    c.jacobi_sweeps += hs[2];
    if (c.o.verbose >= 2) fprintf(stderr, "    jacobi(coop) p=%ld q=%d sweeps %u\n", (long)p, q, hs[2]);
    return;
  }
  for (int sweep = 0; sweep < 40; ++sweep) {
    c.jacobi_sweeps++;
    VSIE_CHECK_CUDA(cudaMemsetAsync(c.ws.rotcnt.p, 0, sizeof(unsigned), c.st));
    for (int t = 0; t < Q - 1; ++t)
      launch_jacobi_round(A, p, p, V, q, sch + (int64_t)t * (Q / 2), Q / 2, thr, small2, c.ws.rotcnt.p, c.st);
    unsigned cnt = 0;
    VSIE_CHECK_CUDA(cudaMemcpyAsync(&cnt, c.ws.rotcnt.p, sizeof(unsigned), cudaMemcpyDeviceToHost, c.st));
    sync(c);
    if (c.o.verbose >= 2) fprintf(stderr, "    jacobi p=%ld q=%d sweep %d rotations %u\n", (long)p, q, sweep, cnt);
    if (cnt == 0) return;
  }
}

// column norms of A (p x q), sorted descending: (sigma, column)
std::vector<std::pair<double, int>> sorted_norms(Ctx& c, const cplx* A, int64_t p, int q) {
  c.ws.norms.ensure(q);
  launch_col_norms(A, p, q, p, c.ws.norms.p, c.st);
  std::vector<double> s(q);
  VSIE_CHECK_CUDA(cudaMemcpyAsync(s.data(), c.ws.norms.p, q * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  std::vector<std::pair<double, int>> v(q);
  for (int j = 0; j < q; ++j) v[j] = {s[j], j};
  std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  return v;
}

// Truncation rule: smallest r with ||sigma[r:]||_2 <= delta ||M||_F.
// randomized: the sketch may miss mass, so the tail is also bounded by ||M||_F^2 - head.
int choose_rank(const std::vector<std::pair<double, int>>& s, double total2, bool randomized, double delta, int cap) {
  const int q = (int)s.size();
  std::vector<double> tail(q + 1, 0.0);
  for (int j = q - 1; j >= 0; --j) tail[j] = tail[j + 1] + s[j].first * s[j].first;
  double head = 0;
  const double lim2 = delta * delta * total2;
  for (int r = 1; r <= q; ++r) {
    head += s[r - 1].first * s[r - 1].first;
    double t2 = tail[r];
    if (randomized) t2 = std::max(t2, total2 - head);
    if (t2 <= lim2) return std::min(r, cap);
  }
  return std::min(q, cap);
}

void upload_idx(Ctx& c, const std::vector<int>& v) {
  c.ws.idx.ensure(std::max<size_t>(1, v.size()));
  VSIE_CHECK_CUDA(cudaMemcpyAsync(c.ws.idx.p, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
}

void zgemm1(Ctx& c, Trans ta, Trans tb, int64_t M, int64_t N, int64_t K, const cplx* A, int64_t lda, const cplx* B,
            int64_t ldb, cplx* C, int64_t ldc) {
  Zgemm z{};
  z.nbatch = 1;
  z.ta = ta;
  z.tb = tb;
  z.M[0] = M; z.N[0] = N; z.K[0] = K;
  z.A[0] = A; z.lda[0] = lda;
  z.B[0] = B; z.ldb[0] = ldb;
  z.C[0] = C; z.ldc[0] = ldc;
  if (!c.ws.zws.p) c.ws.zws.alloc((size_t)16 << 20);  // split-K partials (256 MiB)
  launch_zgemm(z, c.ws.zws.p, (int64_t)c.ws.zws.n, c.st);
}

// C = op(A) B on the FP64 tensor cores (3M DMMA, linalg.cu) for the large products of the
// range finder; op(A) = A^H is computed as conj(A^T conj(B)) (conj(B) staged in ws.Bc)
void zgemm_tc(Ctx& c, Trans ta, int64_t M, int64_t N, int64_t K, const cplx* A, int64_t lda, const cplx* B,
              int64_t ldb, cplx* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  if (!c.ws.zws.p) c.ws.zws.alloc((size_t)16 << 20);
  const cplx* Bu = B;
  int64_t ldbu = ldb;
  if (ta == kC) {
    c.ws.Bc.ensure(K * N);
    launch_copy_conj(B, ldb, K, N, c.ws.Bc.p, c.st);
    Bu = c.ws.Bc.p;
    ldbu = K;
  }
  Zgemm z{};
  z.nbatch = 1;
  z.ta = ta == kC ? kT : ta;
  z.tb = kN;
  z.M[0] = M; z.N[0] = N; z.K[0] = K;
  z.A[0] = A; z.lda[0] = lda;
  z.B[0] = Bu; z.ldb[0] = ldbu;
  z.C[0] = C; z.ldc[0] = ldc;
  launch_zgemm_dmma(z, c.ws.zws.p, (int64_t)c.ws.zws.n, c.st);
  if (ta == kC) launch_conj_2d(C, ldc, M, N, c.st);
}

// ---- row-split helpers of the multi-process build
void rank_rows(const Ctx& c, int64_t rows, int p, int64_t& r0, int64_t& r1) {
  const int P = c.h->world;
  r0 = rows * p / P;
  r1 = rows * (p + 1) / P;
}

// every rank holds rows [r0_p, r1_p) of a rows x ncols matrix (local, ld r1_p - r0_p):
// full (rows x ncols, ld rows) on every rank (allgather of equal padded blocks)
void assemble_rows(Ctx& c, const cplx* local, int64_t rows, int64_t ncols, cplx* full) {
  vsie_coupling_s* h = c.h;
  const int P = h->world;
  const int64_t rpmax = ceil_div(rows, P);
  int64_t r0, r1;
  rank_rows(c, rows, h->rank, r0, r1);
  c.ws.gsend.ensure(std::max<int64_t>(1, rpmax * ncols));
  c.ws.grecv.ensure(std::max<int64_t>(1, P * rpmax * ncols));
  if (r1 > r0)
    VSIE_CHECK_CUDA(cudaMemcpy2DAsync(c.ws.gsend.p, rpmax * sizeof(cplx), local, (r1 - r0) * sizeof(cplx),
                                      (r1 - r0) * sizeof(cplx), ncols, cudaMemcpyDeviceToDevice, c.st));
  h->comm->allgather(reinterpret_cast<const double*>(c.ws.gsend.p), reinterpret_cast<double*>(c.ws.grecv.p),
                     2 * (size_t)(rpmax * ncols), c.st);
  for (int p = 0; p < P; ++p) {
    int64_t a, b;
    rank_rows(c, rows, p, a, b);
    if (b > a)
      VSIE_CHECK_CUDA(cudaMemcpy2DAsync(full + a, rows * sizeof(cplx), c.ws.grecv.p + (int64_t)p * rpmax * ncols,
                                        rpmax * sizeof(cplx), (b - a) * sizeof(cplx), ncols,
                                        cudaMemcpyDeviceToDevice, c.st));
  }
}

void allreduce_c(Ctx& c, cplx* buf, int64_t n) {
  c.h->comm->allreduce_sum(reinterpret_cast<double*>(buf), 2 * (size_t)n, c.st);
}

void set_identity(Ctx& c, DevBuf<cplx>& V, int q) {
  V.ensure((int64_t)q * q);
  std::vector<cplx> I((size_t)q * q, cmk(0, 0));
  for (int j = 0; j < q; ++j) I[(size_t)j * q + j] = cmk(1, 0);
  VSIE_CHECK_CUDA(cudaMemcpyAsync(V.p, I.data(), I.size() * sizeof(cplx), cudaMemcpyHostToDevice, c.st));
  sync(c);
}

// Gram-preconditioned one-sided Jacobi SVD of a tall A (p x q): the eigenvectors
// V1 of G = A^H A (one-sided Jacobi on the q x q Cholesky factor of G + s I; the
// shift only guards the factorisation, eigenvectors are unchanged) make the
// columns of A V1 orthogonal except among singular values below sqrt(u) ||A||,
// so the final one-sided Jacobi on the tall A V1 converges in a few sweeps while
// keeping the one-sided method's relative accuracy.  On exit A holds U S and
// V (if given) the accumulated right singular vectors V1 V2.
void precond_jacobi(Ctx& c, cplx* A, int64_t p, int q, cplx* V, double small_rel = 1e-14) {
  Ws& w = c.ws;
  if (q <= 1) {
    if (V) {
      set_identity(c, w.Rtmp, 1);
      VSIE_CHECK_CUDA(cudaMemcpyAsync(V, w.Rtmp.p, sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
    }
    return;
  }
  const int64_t qq = (int64_t)q * q;
  w.G.ensure(qq);
  w.Rtmp.ensure(qq);
  w.Atmp.ensure(p * q);
  w.frob.ensure(1);
  w.bad.ensure(1);
  VSIE_CHECK_CUDA(cudaMemsetAsync(w.bad.p, 0, sizeof(int), c.st));
  auto t0 = Clock::now();
  zgemm1(c, kC, kN, q, q, p, A, p, A, p, w.G.p, q);
  launch_trace_real(w.G.p, q, w.frob.p, c.st);
  double tr = 0;
  VSIE_CHECK_CUDA(cudaMemcpyAsync(&tr, w.frob.p, sizeof(double), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  if (!(tr > 0)) {
    if (V) {
      set_identity(c, w.Rtmp, q);
      VSIE_CHECK_CUDA(cudaMemcpyAsync(V, w.Rtmp.p, qq * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
    }
    return;
  }
  t0 = Clock::now();
  launch_add_diag(w.G.p, q, 1e-13 * tr, c.st);
  launch_cholesky_upper(w.G.p, q, w.bad.p, c.st);
  int bad = 0;
  VSIE_CHECK_CUDA(cudaMemcpyAsync(&bad, w.bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  c.t_chol += secs(t0);
  set_identity(c, w.Ra, q);
  cplx* V1 = w.Ra.p;
  if (!bad) {
    t0 = Clock::now();
    jacobi(c, w.G.p, q, q, V1, small_rel);  // G now holds R V1 (not needed)
    c.t_jsmall += secs(t0);
    t0 = Clock::now();
    zgemm1(c, kN, kN, p, q, q, A, p, V1, q, w.Atmp.p, p);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(A, w.Atmp.p, p * q * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
    sync(c);
    c.t_gemm += secs(t0);
  }
  w.Rb.ensure(qq);
  set_identity(c, w.Rb, q);
  t0 = Clock::now();
  jacobi(c, A, p, q, w.Rb.p, small_rel);
  if (V) zgemm1(c, kN, kN, q, q, q, V1, q, w.Rb.p, q, V, q);
}

// SVD of a tall A (p x q) with Jacobi sweeps only over the small q x q factor (the large
// factorisations of the randomized range finder: the tall one-sided Jacobi of precond_jacobi
// was 87% of the round-1 cfg 3 build; Gram-based CholeskyQR cannot resolve the singular values
// near 1e-8 of the largest that the cfg 3 truncation needs):
//   1. blocked Householder QR A = Q R (hqr.cu; backward stable for any rank / condition);
//   2. want_svd: one-sided Jacobi on R: R V = U_R S, A <- Q [U_R S; 0] = U S (precond_jacobi's
//      contract: columns U S, unsorted, V the right singular vectors);
//      else A <- Q [I; 0] (orthonormal columns spanning A's range).
void svd_hqr(Ctx& c, cplx* A, int64_t p, int q, cplx* V, bool want_svd) {
  Ws& w = c.ws;
  const int64_t qq = (int64_t)q * q;
  const int pw = hqr_panel_width();
  w.tau.ensure(q);
  w.Th.ensure((size_t)hqr_panels(q) * pw * pw);
  w.Vh.ensure(p * pw);
  w.W.ensure((int64_t)pw * q);
  w.W2.ensure((int64_t)pw * q);
  w.Gv.ensure((int64_t)pw * pw);
  w.hpart.ensure(hqr_part_doubles());
  w.G.ensure(qq);
  w.Atmp.ensure(p * q);
  if (!c.ws.zws.p) c.ws.zws.alloc((size_t)16 << 20);
  const HqrWs hw{w.Vh.p, w.W.p, w.W2.p, w.Gv.p, w.hpart.p, w.zws.p, (int64_t)w.zws.n};
  auto t0 = Clock::now();
  hqr_factor(A, p, p, q, w.tau.p, w.Th.p, hw, c.st);
  sync(c);
  c.t_chol += secs(t0);
  if (want_svd) {
    t0 = Clock::now();
    hqr_copy_r(A, p, q, w.G.p, c.st);
    set_identity(c, w.Rtmp, q);
    cplx* Vq = V ? V : w.Rtmp.p;
    if (V) VSIE_CHECK_CUDA(cudaMemcpyAsync(V, w.Rtmp.p, qq * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
    jacobi(c, w.G.p, q, q, Vq);   // R <- U_R S
    c.t_jsmall += secs(t0);
    hqr_fill(w.G.p, q, q, p, q, w.Atmp.p, p, false, c.st);
  } else {
    hqr_fill(nullptr, 0, q, p, q, w.Atmp.p, p, true, c.st);
  }
  t0 = Clock::now();
  hqr_apply_q(A, p, p, q, w.Th.p, w.Atmp.p, p, q, hw, c.st);
  VSIE_CHECK_CUDA(cudaMemcpyAsync(A, w.Atmp.p, p * q * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
  sync(c);
  c.t_gemm += secs(t0);
}

// the tall SVD used by the factorisations: Householder + small Jacobi for wide factors,
// the preconditioned tall Jacobi for q <= 384 (cheap there, and proven since round 1)
void tall_svd(Ctx& c, cplx* A, int64_t p, int q, cplx* V) {
  if (q > 384 && p >= q)
    svd_hqr(c, A, p, q, V, true);
  else
    precond_jacobi(c, A, p, q, V);
}

// Rank-revealing factorisation of M (rows x cols, ld rows).
//  left = true : ws.basis <- rows x r basis of the dominant column space (L of L->R)
//  left = false: ws.basis <- cols x r basis R with M ~ X R^T (R->L)
// other != null also receives the basis of the opposite side (right basis R for
// left = true, left basis L for left = false) of the same truncated SVD, so that
// the half-sweep turnaround on the same supercore needs no second factorisation.
// Multi-process (c.dist): M holds this rank's rows [c.rp0, c.rp1) (ld rp1 - rp0) of the
// rows x cols supercore; small supercores are assembled and factorised on every rank, the
// randomized path keeps M row-split: the sketch M Omega is formed locally and allgathered
// (L->R) or its sum M^H Omega = sum_p M_p^H Omega_p allreduced (R->L), B = Q^H M likewise --
// no rank ever holds the whole large supercore; the small factorisations are replicated
// (bitwise identical inputs on every rank, so every rank picks the same ranks and pivots).
int factorize(Ctx& c, const cplx* M, int64_t rows, int64_t cols, bool left, int r_prev, DevBuf<cplx>* other) {
  Ws& w = c.ws;
  const int64_t mn = std::min(rows, cols);
  const int cap = (int)std::min<int64_t>(c.o.max_rank, mn);
  const int64_t rl = c.dist ? c.rp1 - c.rp0 : rows;   // local rows of M
  if (c.dist && mn <= c.o.direct_svd_max) {
    w.Mfull.ensure(rows * cols);
    assemble_rows(c, M, rows, cols, w.Mfull.p);
    M = w.Mfull.p;
  }
  if (mn <= c.o.direct_svd_max) {
    const bool tall = rows >= cols;
    const int64_t p = tall ? rows : cols;
    const int q = (int)(tall ? cols : rows);
    w.J.ensure(p * q);
    if (tall)
      VSIE_CHECK_CUDA(cudaMemcpyAsync(w.J.p, M, p * q * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
    else
      launch_transpose(M, rows, cols, w.J.p, true, c.st);  // M^H
    w.V.ensure((int64_t)q * q);
    precond_jacobi(c, w.J.p, p, q, w.V.p);
    auto s = sorted_norms(c, w.J.p, p, q);
    double total2 = 0;
    for (auto& e : s) total2 += e.first * e.first;
    int r = total2 > 0 ? choose_rank(s, total2, false, c.delta, cap) : 1;
    std::vector<int> sel(r);
    for (int j = 0; j < r; ++j) sel[j] = s[j].second;
    upload_idx(c, sel);
    if (left) {
      w.basis.ensure(rows * r);
      if (tall)
        launch_gather_cols(w.J.p, rows, rows, c.ws.idx.p, nullptr, r, w.basis.p, rows, false, c.st);
      else
        launch_gather_cols(w.V.p, rows, q, c.ws.idx.p, nullptr, r, w.basis.p, rows, false, c.st);
    } else {
      w.basis.ensure(cols * r);
      if (tall)
        launch_gather_cols(w.V.p, cols, q, c.ws.idx.p, nullptr, r, w.basis.p, cols, true, c.st);
      else
        launch_gather_cols(w.J.p, cols, cols, c.ws.idx.p, nullptr, r, w.basis.p, cols, true, c.st);
    }
    if (other) {
      if (left) {  // right basis conj(V_sel) (tall) or conj(M^H V_sel) (wide)
        other->ensure(cols * r);
        if (tall)
          launch_gather_cols(w.V.p, cols, q, c.ws.idx.p, nullptr, r, other->p, cols, true, c.st);
        else
          launch_gather_cols(w.J.p, cols, cols, c.ws.idx.p, nullptr, r, other->p, cols, true, c.st);
      } else {     // left basis M V_sel (tall) or V_sel (wide)
        other->ensure(rows * r);
        if (tall)
          launch_gather_cols(w.J.p, rows, rows, c.ws.idx.p, nullptr, r, other->p, rows, false, c.st);
        else
          launch_gather_cols(w.V.p, rows, q, c.ws.idx.p, nullptr, r, other->p, rows, false, c.st);
      }
    }
    return r;
  }
  // ---- randomized range finder (SURVEY §8c-X GPU-scale variant, no power iteration)
  const int os = c.o.oversample;
  w.frob_partial.ensure(1024);
  w.frob.ensure(1);
  launch_frob2(M, rl * cols, w.frob_partial.p, w.frob.p, c.st);
  if (c.dist) c.h->comm->allreduce_sum(w.frob.p, 1, c.st);
  double total2 = 0;
  VSIE_CHECK_CUDA(cudaMemcpyAsync(&total2, w.frob.p, sizeof(double), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  if (!(total2 > 0)) {
    // zero supercore: rank 1 with a unit basis vector
    const int64_t n = left ? rows : cols;
    w.basis.ensure(n);
    VSIE_CHECK_CUDA(cudaMemsetAsync(w.basis.p, 0, n * sizeof(cplx), c.st));
    const cplx one = cmk(1, 0);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(w.basis.p, &one, sizeof(cplx), cudaMemcpyHostToDevice, c.st));
    sync(c);
    return 1;
  }
  int kk = (int)std::min<int64_t>(std::max(r_prev, 1) + os, mn);
  const int64_t p1 = left ? rows : cols, p2 = left ? cols : rows;
  int kk_done = 0;   // columns of the raw sketch already formed (a grown sketch keeps them)
  for (;;) {
    // Y = M Omega (L->R) or M^H Omega (R->L) for the new columns [kk_done, kk): a Gaussian Omega
    // per column block; R->L as conj(M^T Omega) = M^H conj(Omega), an equally Gaussian sketch
    {
      const int nn = kk - kk_done;
      w.omega.ensure(p2 * nn);
      launch_gaussian(w.omega.p, p2 * nn, c.seed ^ (0xABCDEF12345ull + 977 * (++c.sketch_counter)), c.st);
      if (kk_done == 0) {
        w.Yraw.ensure(p1 * (int64_t)std::min<int64_t>(mn, 2 * (int64_t)kk + 4 * os));
      } else if ((int64_t)w.Yraw.n < p1 * kk) {
        DevBuf<cplx> grown(p1 * (int64_t)std::min<int64_t>(mn, 2 * (int64_t)kk + 4 * os));
        VSIE_CHECK_CUDA(cudaMemcpyAsync(grown.p, w.Yraw.p, p1 * kk_done * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
        sync(c);
        w.Yraw = std::move(grown);
      }
      cplx* dst = w.Yraw.p + p1 * kk_done;
      if (left) {
        if (c.dist) {   // local rows of M Omega, allgathered into the full sketch
          w.Yloc.ensure(std::max<int64_t>(1, rl * nn));
          zgemm_tc(c, kN, rl, nn, cols, M, rl, w.omega.p, cols, w.Yloc.p, rl);
          assemble_rows(c, w.Yloc.p, rows, nn, dst);
        } else {
          zgemm_tc(c, kN, rows, nn, cols, M, rows, w.omega.p, cols, dst, rows);
        }
      } else {
        // conj(M^T Omega) = M^H conj(Omega); row-split: sum over the ranks' row blocks
        zgemm_tc(c, kT, cols, nn, rl, M, rl, w.omega.p + (c.dist ? c.rp0 : 0), rows, dst, cols);
        if (c.dist) allreduce_c(c, dst, cols * nn);
        launch_conj(dst, p1 * nn, c.st);
      }
      kk_done = kk;
    }
    w.Y.ensure(p1 * kk);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(w.Y.p, w.Yraw.p, p1 * kk * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
    // Orthonormal basis Q of the sketch's range: Householder QR (unit columns; for a rank-
    // deficient sketch the extra columns are orthonormal directions with ~zero weight in B
    // below).  The preconditioned tall Jacobi -- which leaves directions below 1e-3 delta
    // ||Y||_F unrotated -- measured slower even on the narrow 576k-row sketches of the cfg 3
    // R->L k = 2 supercore (157 vs 125 s for the cfg 3 build).
    const bool hq = true;
    svd_hqr(c, w.Y.p, p1, kk, nullptr, false);   // kk <= mn <= p1
    auto sy = sorted_norms(c, w.Y.p, p1, kk);
    const double cut = 0.5 * sy[0].first;   // unit columns
    (void)hq;
    std::vector<int> keep;
    std::vector<double> inv;
    for (auto& e : sy)
      if (e.first > cut) {
        keep.push_back(e.second);
        inv.push_back(1.0 / e.first);
      }
    const int kq = (int)keep.size();
    upload_idx(c, keep);
    w.norms.ensure(std::max(kq, kk));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(w.norms.p, inv.data(), kq * sizeof(double), cudaMemcpyHostToDevice, c.st));
    w.Q.ensure(p1 * kq);
    launch_gather_cols(w.Y.p, p1, p1, c.ws.idx.p, w.norms.p, kq, w.Q.p, p1, false, c.st);
    // Bh = M^H Q (L->R) or M Q (R->L): p2 x kq
    w.Bh.ensure(p2 * kq);
    if (left) {   // M^H Q = sum over the row blocks M_p^H Q_p
      zgemm_tc(c, kC, cols, kq, rl, M, rl, w.Q.p + (c.dist ? c.rp0 : 0), rows, w.Bh.p, cols);
      if (c.dist) allreduce_c(c, w.Bh.p, cols * kq);
    } else if (c.dist) {   // M Q: local rows, allgathered
      w.Bloc.ensure(std::max<int64_t>(1, rl * kq));
      zgemm_tc(c, kN, rl, kq, cols, M, rl, w.Q.p, cols, w.Bloc.p, rl);
      assemble_rows(c, w.Bloc.p, rows, kq, w.Bh.p);
    } else {
      zgemm_tc(c, kN, rows, kq, cols, M, rows, w.Q.p, cols, w.Bh.p, rows);
    }
    w.V.ensure((int64_t)kq * kq);
    tall_svd(c, w.Bh.p, p2, kq, w.V.p);
    auto s = sorted_norms(c, w.Bh.p, p2, kq);
    int nnz = 0;   // exactly zero singular values are never part of a basis
    for (auto& e : s) nnz += e.first > 0 ? 1 : 0;
    const int r = choose_rank(s, total2, true, c.delta, std::max(1, std::min({cap, kq, nnz})));
    // grow the sketch while the rank leaves less than `os` oversampling inside it (a sketch
    // whose range is exhausted -- kq well below kk -- already holds M's numerical range)
    if (r > kq - os && kq > kk - os && kk < mn) {
      // rank found inside the sketch but with less than `os` oversampling: grow to
      // r + 2 os (a rank drift of a few per sweep no longer doubles a ~300-column sketch,
      // whose Jacobi cost grows as q^2); a saturated sketch (r == kq) doubles
      const int64_t grow = r < kq ? (int64_t)r + 2 * os : 2 * (int64_t)kk;
      kk = (int)std::min<int64_t>(std::max<int64_t>(grow, (int64_t)kk + os), mn);
      continue;
    }
    std::vector<int> sel(r);
    for (int j = 0; j < r; ++j) sel[j] = s[j].second;
    upload_idx(c, sel);
    w.Vr.ensure((int64_t)kq * r);
    launch_gather_cols(w.V.p, kq, kq, c.ws.idx.p, nullptr, r, w.Vr.p, kq, false, c.st);
    w.basis.ensure(p1 * r);
    zgemm1(c, kN, kN, p1, r, kq, w.Q.p, p1, w.Vr.p, kq, w.basis.p, p1);
    if (!left) launch_conj(w.basis.p, p1 * r, c.st);
    if (other) {  // Bh V = U S: conj for the right basis (L->R), as is for the left basis (R->L)
      other->ensure(p2 * r);
      launch_gather_cols(w.Bh.p, p2, p2, c.ws.idx.p, nullptr, r, other->p, p2, left, c.st);
    }
    return r;
  }
}

// maxvol on A (n x r, destroyed): returns pivot rows (original order) and
// Bout = A A[P]^{-1} (n x r).
std::vector<int> maxvol(Ctx& c, cplx* A, int64_t n, int r, cplx* Bout) {
  Ws& w = c.ws;
  const int nparts = lu_nparts(n);
  w.partials.ensure(nparts);
  w.perm.ensure(n);
  w.bad.ensure(1);
  {
    std::vector<int> iota(n);
    std::iota(iota.begin(), iota.end(), 0);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(w.perm.p, iota.data(), n * sizeof(int), cudaMemcpyHostToDevice, c.st));
    VSIE_CHECK_CUDA(cudaMemsetAsync(w.bad.p, 0, sizeof(int), c.st));
  }
  // 1. initial pivots: LU with partial pivoting (rows physically swapped)
  const auto t_lu = Clock::now();
  // blocked right-looking: per panel of kLuPanel columns the unblocked steps restricted to the
  // panel, then U12 = L11^{-1} A12 and A22 -= L21 U12 (one ZGEMM) -- the same pivots as the
  // column-by-column LU up to the rounding order of the trailing updates, at n r^2 / kLuPanel
  // instead of n r^2 bytes of rank-1 update traffic
  launch_lu_update(A, n, r, -1, r, false, true, w.partials.p, nparts, c.st);
  for (int j0 = 0; j0 < r; j0 += kLuPanel) {
    const int jb = std::min(kLuPanel, r - j0);
    for (int j = j0; j < j0 + jb; ++j) {
      launch_lu_pivot(A, n, r, j, w.perm.p, w.partials.p, nparts, w.bad.p, c.st);
      launch_lu_update(A, n, r, j, j0 + jb, true, j + 1 < j0 + jb, w.partials.p, nparts, c.st);
    }
    if (j0 + jb < r) {
      launch_lu_trsm(A, n, r, j0, jb, c.st);
      Zgemm z{};
      z.nbatch = 1;
      z.ta = kN;
      z.tb = kN;
      z.M[0] = n - j0 - jb;
      z.N[0] = r - j0 - jb;
      z.K[0] = jb;
      z.A[0] = A + (j0 + jb) + n * j0;
      z.lda[0] = n;
      z.B[0] = A + j0 + n * (j0 + jb);
      z.ldb[0] = n;
      z.C[0] = A + (j0 + jb) + n * (j0 + jb);
      z.ldc[0] = n;
      z.alpha = cmk(-1, 0);
      z.beta = cmk(1, 0);
      if (z.M[0] > 0) launch_zgemm(z, nullptr, 0, c.st);
      launch_lu_update(A, n, r, j0 + jb - 1, r, false, true, w.partials.p, nparts, c.st);   // next pivot column
    }
  }
  int bad = 0;
  VSIE_CHECK_CUDA(cudaMemcpyAsync(&bad, w.bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  c.t_maxvol_lu += secs(t_lu);
  VSIE_REQUIRE(!bad, VSIE_ERR_CUDA, "maxvol: rank-deficient factor (zero pivot in LU)");
  // 2. B_perm = [I_r ; L2 L1^{-1}]
  w.Lr.ensure((int64_t)r * r);
  w.T.ensure((int64_t)r * r);
  launch_copy_lower(A, n, r, w.Lr.p, c.st);
  launch_unit_lower_inverse(w.Lr.p, r, w.T.p, c.st);
  w.Bp.ensure(n * r);
  launch_set_identity_top(w.Bp.p, n, r, c.st);
  if (n > r) zgemm1(c, kN, kN, n - r, r, r, A + r, n, w.T.p, r, w.Bp.p + r, n);
  // 3. swaps while max |B| > 1 + tau
  w.piv_pos.ensure(r);
  w.rowbuf.ensure(r);
  w.mvs.ensure(1);
  {
    std::vector<int> iota(r);
    std::iota(iota.begin(), iota.end(), 0);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(w.piv_pos.p, iota.data(), r * sizeof(int), cudaMemcpyHostToDevice, c.st));
    VSIE_CHECK_CUDA(cudaMemsetAsync(w.mvs.p, 0, sizeof(MaxvolState), c.st));
  }
  const double tau = 0.05;
  launch_maxvol_update(w.Bp.p, n, r, w.perm.p, w.rowbuf.p, w.mvs.p, false, w.partials.p, nparts, c.st);
  const int it_max = 100 * r;
  int it = 0;
  MaxvolState hs{};
  while (it < it_max) {
    const int batch = std::min(16, it_max - it);
    for (int b = 0; b < batch; ++b) {
      launch_maxvol_select(w.Bp.p, n, r, w.partials.p, nparts, tau, w.piv_pos.p, w.rowbuf.p, w.mvs.p, c.st);
      launch_maxvol_update(w.Bp.p, n, r, w.perm.p, w.rowbuf.p, w.mvs.p, true, w.partials.p, nparts, c.st);
    }
    it += batch;
    VSIE_CHECK_CUDA(cudaMemcpyAsync(&hs, w.mvs.p, sizeof(MaxvolState), cudaMemcpyDeviceToHost, c.st));
    sync(c);
    if (hs.done) break;
  }
  c.maxvol_swaps += hs.swaps;
  // 4. outputs in the original row order
  std::vector<int> perm(n), pos(r), piv(r);
  VSIE_CHECK_CUDA(cudaMemcpyAsync(perm.data(), w.perm.p, n * sizeof(int), cudaMemcpyDeviceToHost, c.st));
  VSIE_CHECK_CUDA(cudaMemcpyAsync(pos.data(), w.piv_pos.p, r * sizeof(int), cudaMemcpyDeviceToHost, c.st));
  launch_scatter_rows(w.Bp.p, n, r, w.perm.p, Bout, c.st);
  sync(c);
  for (int j = 0; j < r; ++j) piv[j] = perm[pos[j]];
  return piv;
}

// ------------------------------------------------------------------ per-chi cross state
struct ChiState {
  int chi;
  int r[5] = {1, 1, 1, 1, 1};
  std::vector<std::array<int, 1>> I1;
  std::vector<std::array<int, 2>> I2;
  std::vector<std::array<int, 3>> I3;
  std::vector<std::array<int, 3>> J1;  // (i2, i3, n)
  std::vector<std::array<int, 2>> J2;  // (i3, n)
  std::vector<std::array<int, 1>> J3;  // (n)
  DevBuf<cplx> core[4];
};

int dim(const vsie_coupling_s* h, int k) { return k < 3 ? h->grid.n[k] : (int)h->m; }

// Evaluates M_k into ws.M (rows x cols, ld rows); column blocks split across NCCL ranks.
void eval_supercore(Ctx& c, ChiState& s, int k, int64_t& rows, int64_t& cols) {
  vsie_coupling_s* h = c.h;
  const int64_t rl = s.r[k - 1], nk = dim(h, k - 1), nk1 = dim(h, k), rr = s.r[k + 1];
  rows = rl * nk;
  cols = nk1 * rr;
  std::vector<int32_t> left(2 * std::max<int64_t>(rl, 1), 0), right(2 * std::max<int64_t>(rr, 1), 0);
  if (k == 2)
    for (int64_t a = 0; a < rl; ++a) left[2 * a] = s.I1[a][0];
  if (k == 3)
    for (int64_t a = 0; a < rl; ++a) { left[2 * a] = s.I2[a][0]; left[2 * a + 1] = s.I2[a][1]; }
  if (k == 1)
    for (int64_t b = 0; b < rr; ++b) { right[2 * b] = s.J2[b][0]; right[2 * b + 1] = s.J2[b][1]; }
  if (k == 2)
    for (int64_t b = 0; b < rr; ++b) right[2 * b] = s.J3[b][0];
  c.ws.left.ensure(left.size());
  c.ws.right.ensure(right.size());
  VSIE_CHECK_CUDA(cudaMemcpyAsync(c.ws.left.p, left.data(), left.size() * 4, cudaMemcpyHostToDevice, c.st));
  VSIE_CHECK_CUDA(cudaMemcpyAsync(c.ws.right.p, right.data(), right.size() * 4, cudaMemcpyHostToDevice, c.st));
  c.dist = h->comm != nullptr;
  c.rp0 = 0;
  c.rp1 = rows;
  if (c.dist) rank_rows(c, rows, h->rank, c.rp0, c.rp1);   // this rank's rows
  c.ws.M.ensure(std::max<int64_t>(1, (c.rp1 - c.rp0) * cols));
  BlockDesc b{};
  b.chi = s.chi;
  b.k = k;
  b.rl = rl; b.nk = nk; b.nk1 = nk1; b.rr = rr;
  b.left = c.ws.left.p;
  b.right = c.ws.right.p;
  b.ld = c.rp1 - c.rp0;
  b.col0 = 0;
  b.col1 = cols;
  b.row0 = c.rp0;
  b.row1 = c.rp1;
  auto t0 = Clock::now();
  if (c.rp1 > c.rp0) launch_entries_block(h->eg, b, c.ws.M.p, c.st);
  sync(c);
  c.t_entry += secs(t0);
  c.n_eval += rows * cols;
}

// held-out sample (seeded) and exact values
struct Heldout {
  std::vector<std::array<int, 4>> idx;
  std::vector<cplx> exact;
  DevBuf<int64_t> d_idx;
  DevBuf<cplx> d_out;
};

bool on_cross(const ChiState& s, const std::array<int, 4>& t) {
  auto in1 = [&](const auto& set, auto key) { return std::find(set.begin(), set.end(), key) != set.end(); };
  if (in1(s.I1, std::array<int, 1>{t[0]}) && in1(s.J1, std::array<int, 3>{t[1], t[2], t[3]})) return true;
  if (in1(s.I2, std::array<int, 2>{t[0], t[1]}) && in1(s.J2, std::array<int, 2>{t[2], t[3]})) return true;
  if (in1(s.I3, std::array<int, 3>{t[0], t[1], t[2]}) && in1(s.J3, std::array<int, 1>{t[3]})) return true;
  return false;
}

double heldout_error(Ctx& c, ChiState& s, Heldout& ho) {
  vsie_coupling_s* h = c.h;
  const int n[3] = {h->grid.n[0], h->grid.n[1], h->grid.n[2]};
  const cplx* G[4] = {s.core[0].p, s.core[1].p, s.core[2].p, s.core[3].p};
  const int r[3] = {s.r[1], s.r[2], s.r[3]};
  const int64_t cnt = (int64_t)ho.idx.size();
  launch_tt_eval(G, r, n, h->m, s.chi, ho.d_idx.p, cnt, h->grid.nv(), ho.d_out.p, c.st);
  std::vector<cplx> tt(cnt);
  VSIE_CHECK_CUDA(cudaMemcpyAsync(tt.data(), ho.d_out.p, cnt * sizeof(cplx), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  double num = 0, den = 0;
  for (int64_t i = 0; i < cnt; ++i) {
    if (on_cross(s, ho.idx[i])) continue;
    const cplx d = csub(tt[i], ho.exact[i]);
    num += cabs2(d);
    den += cabs2(ho.exact[i]);
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

void copy_core(DevBuf<cplx>& dst, const DevBuf<cplx>& src, size_t n, cudaStream_t st) {
  dst.ensure(n);
  VSIE_CHECK_CUDA(cudaMemcpyAsync(dst.p, src.p, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
}

size_t core_elems(const vsie_coupling_s* h, const int r[5], int k) {
  return (size_t)r[k] * dim(h, k) * r[k + 1];
}

int cross_chi(Ctx& c, int chi, Heldout& ho) {
  vsie_coupling_s* h = c.h;
  ChiState s;
  s.chi = chi;
  // initial right sets from one seeded index (nested by construction)
  uint64_t rs = c.seed + (uint64_t)chi * 1000003ull;
  const int st[4] = {(int)(host_splitmix(rs) % dim(h, 0)), (int)(host_splitmix(rs) % dim(h, 1)),
                     (int)(host_splitmix(rs) % dim(h, 2)), (int)(host_splitmix(rs) % dim(h, 3))};
  s.J3 = {{st[3]}};
  s.J2 = {{st[2], st[3]}};
  s.J1 = {{st[1], st[2], st[3]}};
  // held-out: exact values for this chi
  {
    const int64_t cnt = (int64_t)ho.idx.size();
    std::vector<int64_t> rc(2 * cnt);
    const int64_t nv = h->grid.nv();
    for (int64_t i = 0; i < cnt; ++i) {
      const auto& t = ho.idx[i];
      rc[2 * i] = chi * nv + t[0] + (int64_t)h->grid.n[0] * (t[1] + (int64_t)h->grid.n[1] * t[2]);
      rc[2 * i + 1] = t[3];
    }
    VSIE_CHECK_CUDA(cudaMemcpyAsync(ho.d_idx.p, rc.data(), rc.size() * 8, cudaMemcpyHostToDevice, c.st));
    launch_entries_list(h->eg, ho.d_idx.p, cnt, ho.d_out.p, c.st);
    ho.exact.resize(cnt);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(ho.exact.data(), ho.d_out.p, cnt * sizeof(cplx), cudaMemcpyDeviceToHost, c.st));
    sync(c);
    c.n_eval += cnt;
  }
  DevBuf<cplx> best[4];
  int best_r[5] = {1, 1, 1, 1, 1};
  double best_e = INFINITY;
  int prev[3] = {-1, -1, -1};
  int sweeps = 0;
  bool reuse = false;  // ws.M already holds the next supercore
  int reuse_r = 0;     // ... and ws.other holds its opposite-side basis of rank reuse_r
  int64_t rows = 0, cols = 0;
  for (int sweep = 1; sweep <= c.o.max_sweeps; ++sweep) {
    sweeps = sweep;
    // ---------------- left-to-right
    for (int k = 1; k <= 3; ++k) {
      auto t0 = Clock::now();
      int r;
      if (reuse) {  // same M_1 as the last R->L step: its left basis is ready
        r = reuse_r;
        c.ws.basis.ensure(rows * r);
        VSIE_CHECK_CUDA(cudaMemcpyAsync(c.ws.basis.p, c.ws.other.p, rows * r * sizeof(cplx),
                                        cudaMemcpyDeviceToDevice, c.st));
      } else {
        eval_supercore(c, s, k, rows, cols);
        t0 = Clock::now();
        r = factorize(c, c.ws.M.p, rows, cols, true, s.r[k], k == 3 ? &c.ws.other : nullptr);
      }
      reuse = false;
      sync(c);
      c.t_factor += secs(t0);
      t0 = Clock::now();
      const int rl = s.r[k - 1];
      s.core[k - 1].ensure(rows * r);
      std::vector<int> P = maxvol(c, c.ws.basis.p, rows, r, s.core[k - 1].p);
      c.t_maxvol += secs(t0);
      if (k == 1) {
        s.I1.clear();
        for (int p : P) s.I1.push_back({p});
      } else if (k == 2) {
        s.I2.clear();
        for (int p : P) s.I2.push_back({s.I1[p % rl][0], p / rl});
      } else {
        s.I3.clear();
        for (int p : P) s.I3.push_back({s.I2[p % rl][0], s.I2[p % rl][1], p / rl});
        upload_idx(c, P);
        s.core[3].ensure((int64_t)r * cols);
        if (c.dist) {   // rows P of the row-split M_3: owned rows copied, the rest zero, summed
          launch_gather_rows_owned(c.ws.M.p, c.rp1 - c.rp0, c.ws.idx.p, r, cols, c.rp0, c.rp1, s.core[3].p, c.st);
          allreduce_c(c, s.core[3].p, (int64_t)r * cols);
        } else {
          launch_gather_rows(c.ws.M.p, rows, c.ws.idx.p, r, cols, s.core[3].p, c.st);
        }
        reuse = true;  // R->L starts with the same M_3 (right basis in ws.other)
        reuse_r = r;
      }
      s.r[k] = r;
    }
    // ---------------- right-to-left
    for (int k = 3; k >= 1; --k) {
      auto t0 = Clock::now();
      int r;
      if (reuse) {  // same M_3 as the last L->R step: its right basis is ready
        r = reuse_r;
        c.ws.basis.ensure(cols * r);
        VSIE_CHECK_CUDA(cudaMemcpyAsync(c.ws.basis.p, c.ws.other.p, cols * r * sizeof(cplx),
                                        cudaMemcpyDeviceToDevice, c.st));
      } else {
        eval_supercore(c, s, k, rows, cols);
        t0 = Clock::now();
        r = factorize(c, c.ws.M.p, rows, cols, false, s.r[k], k == 1 ? &c.ws.other : nullptr);
      }
      reuse = false;
      sync(c);
      c.t_factor += secs(t0);
      t0 = Clock::now();
      c.ws.Bout.ensure(cols * r);
      std::vector<int> Q = maxvol(c, c.ws.basis.p, cols, r, c.ws.Bout.p);
      const int64_t nk1 = dim(h, k);
      s.core[k].ensure((int64_t)r * cols);
      launch_transpose(c.ws.Bout.p, cols, r, s.core[k].p, false, c.st);
      c.t_maxvol += secs(t0);
      if (k == 3) {
        s.J3.clear();
        for (int q : Q) s.J3.push_back({q});
      } else if (k == 2) {
        s.J2.clear();
        for (int q : Q) s.J2.push_back({(int)(q % nk1), s.J3[q / nk1][0]});
      } else {
        s.J1.clear();
        for (int q : Q) s.J1.push_back({(int)(q % nk1), s.J2[q / nk1][0], s.J2[q / nk1][1]});
        upload_idx(c, Q);
        s.core[0].ensure(rows * r);
        if (c.dist) {   // columns Q of the row-split M_1, rows assembled from the ranks
          const int64_t rloc = c.rp1 - c.rp0;
          c.ws.Bloc.ensure(std::max<int64_t>(1, rloc * r));
          launch_gather_cols(c.ws.M.p, rloc, rloc, c.ws.idx.p, nullptr, r, c.ws.Bloc.p, rloc, false, c.st);
          assemble_rows(c, c.ws.Bloc.p, rows, r, s.core[0].p);
        } else {
          launch_gather_cols(c.ws.M.p, rows, rows, c.ws.idx.p, nullptr, r, s.core[0].p, rows, false, c.st);
        }
        reuse = true;  // the next L->R starts with the same M_1 (left basis in ws.other)
        reuse_r = r;
      }
      s.r[k] = r;
    }
    sync(c);
    const double e = heldout_error(c, s, ho);
    if (c.o.verbose)
      fprintf(stderr, "[vsie cross] chi %d sweep %d ranks (%d, %d, %d) heldout %.3e  (entry %.2fs factor %.2fs [cholqr %.2f jacobi(R) %.2f gemm %.2f] maxvol %.2fs [LU %.2f, %lld swaps], jacobi sweeps %ld)\n",
              chi, sweep, s.r[1], s.r[2], s.r[3], e, c.t_entry, c.t_factor, c.t_chol, c.t_jsmall, c.t_gemm,
              c.t_maxvol, c.t_maxvol_lu, (long long)c.maxvol_swaps, (long)c.jacobi_sweeps);
    if (e < best_e) {
      best_e = e;
      for (int k = 0; k < 5; ++k) best_r[k] = s.r[k];
      for (int k = 0; k < 4; ++k) copy_core(best[k], s.core[k], core_elems(h, s.r, k), c.st);
    }
    // DESIGN.md reading R2: stop when every rank moved by at most max(1, 5%)
    // over the sweep and the held-out error is within the acceptance bound
    bool same = true;
    for (int k = 0; k < 3; ++k) {
      const int d = std::abs(prev[k] - s.r[k + 1]);
      if (prev[k] < 0 || d > std::max(1, s.r[k + 1] / 20)) same = false;
    }
    if (same && e <= 10 * c.tol) break;
    prev[0] = s.r[1];
    prev[1] = s.r[2];
    prev[2] = s.r[3];
  }
  sync(c);
  const int rr[3] = {best_r[1], best_r[2], best_r[3]};
  const cplx* dev[4] = {best[0].p, best[1].p, best[2].p, best[3].p};
  handle_set_cores_device(h, chi, rr, dev);
  h->sweeps[chi] = sweeps;
  h->heldout_err[chi] = best_e;
  return best_e <= 10 * c.tol ? VSIE_OK : VSIE_WARN_NOT_CONVERGED;
}

// ------------------------------------------------------------------ TT rounding
// the cross "might overestimate the TT-ranks";
// rounding = the TT-SVD of the tensor the cores already represent, done on
// the cores (algorithm of the cited [Oseledets 2011]; oracle/ttround.py restates it):
//   1. right-to-left, k = 3..1: core_k^T (as (n_k r_k) x r_{k-1}) = Q R, core_k <- Q^T,
//      core_{k-1} <- core_{k-1} R^T.  Q R comes from the Jacobi SVD X = (X V) V^H:
//      Q = (X V) S^{-1} over the numerically non-zero columns, R = S V^H (so R^T =
//      conj(V) S).  After this ||A||_F = ||core_0||_F.
//   2. left-to-right, k = 0..2: core_k (as (r_{k-1} n_k) x r_k) = U S V^H, keep the
//      smallest r with ||S[r:]|| <= tol / sqrt 3 ||A||_F, core_k <- U_r,
//      core_{k+1} <- S_r V_r^H core_{k+1}.
// cores: full column-major cores of one chi (core_k is r_{k-1} x n_k x r_k); r[0..2] the
// inner ranks; both are replaced.
void round_chi(Ctx& c, const int n[4], int r[3], DevBuf<cplx> core[4]) {
  Ws& w = c.ws;
  int rk[5] = {1, r[0], r[1], r[2], 1};
  // kept columns (and their scales) of a Jacobi-orthogonalised X (p x q, columns U S)
  auto select = [&](const cplx* X, int64_t p, int q, bool truncate, double abs2) {
    auto s = sorted_norms(c, X, p, q);
    int keep;
    if (truncate) {
      keep = q;
      std::vector<double> tail(q + 1, 0.0);
      for (int j = q - 1; j >= 0; --j) tail[j] = tail[j + 1] + s[j].first * s[j].first;
      for (int k = 1; k <= q; ++k)
        if (tail[k] <= abs2) { keep = k; break; }
    } else {
      keep = 0;
      for (auto& e : s)
        if (e.first > 1e-14 * s[0].first) ++keep;
    }
    keep = std::max(keep, 1);
    s.resize(keep);
    return s;
  };
  auto upload_scales = [&](const std::vector<double>& v) {
    w.norms.ensure(std::max<size_t>(1, v.size()));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(w.norms.p, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, c.st));
  };
  DevBuf<cplx> nxt;
  // ---- 1. right-to-left orthogonalisation
  for (int k = 3; k >= 1; --k) {
    const int64_t a = rk[k], nb = (int64_t)n[k] * rk[k + 1];
    const int q = (int)a;
    w.J.ensure(nb * a);
    launch_transpose(core[k].p, a, nb, w.J.p, false, c.st);  // X = core_k^T: (n_k r_k) x r_{k-1}
    w.V.ensure((int64_t)q * q);
    tall_svd(c, w.J.p, nb, q, w.V.p);
    auto s = select(w.J.p, nb, q, false, 0);
    const int rp = (int)s.size();
    if (c.o.verbose)
      fprintf(stderr, "[vsie round] R->L k=%d X %ldx%d kept %d s[0] %.6e s[last] %.6e\n", k, (long)nb, q, rp,
              s[0].first, s.back().first);
    std::vector<int> sel(rp);
    std::vector<double> inv(rp), sv(rp);
    for (int j = 0; j < rp; ++j) {
      sel[j] = s[j].second;
      sv[j] = s[j].first;
      inv[j] = s[j].first > 0 ? 1.0 / s[j].first : 0.0;
    }
    upload_idx(c, sel);
    upload_scales(inv);
    w.Q.ensure(nb * rp);
    launch_gather_cols(w.J.p, nb, nb, c.ws.idx.p, w.norms.p, rp, w.Q.p, nb, false, c.st);  // Q = (X V) S^-1
    nxt.alloc(rp * nb);
    launch_transpose(w.Q.p, nb, rp, nxt.p, false, c.st);                                  // core_k <- Q^T
    std::swap(core[k], nxt);
    upload_scales(sv);
    w.Vr.ensure((int64_t)q * rp);
    launch_gather_cols(w.V.p, q, q, c.ws.idx.p, w.norms.p, rp, w.Vr.p, q, true, c.st);   // R^T = conj(V) S
    const int64_t rows = (int64_t)rk[k - 1] * n[k - 1];
    nxt.alloc(rows * rp);
    zgemm1(c, kN, kN, rows, rp, a, core[k - 1].p, rows, w.Vr.p, q, nxt.p, rows);         // core_{k-1} R^T
    std::swap(core[k - 1], nxt);
    rk[k] = rp;
    sync(c);
  }
  // ---- 2. left-to-right truncation, delta = tol / sqrt(d - 1) ||A||_F, d = 4
  w.frob_partial.ensure(1024);
  w.frob.ensure(1);
  launch_frob2(core[0].p, (int64_t)n[0] * rk[1], w.frob_partial.p, w.frob.p, c.st);
  double nrm2 = 0;
  VSIE_CHECK_CUDA(cudaMemcpyAsync(&nrm2, w.frob.p, sizeof(double), cudaMemcpyDeviceToHost, c.st));
  sync(c);
  const double abs2 = c.tol * c.tol / 3.0 * nrm2;
  for (int k = 0; k < 3; ++k) {
    const int64_t rows = (int64_t)rk[k] * n[k];
    const int q = rk[k + 1];
    w.J.ensure(rows * q);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(w.J.p, core[k].p, rows * q * sizeof(cplx), cudaMemcpyDeviceToDevice, c.st));
    w.V.ensure((int64_t)q * q);
    tall_svd(c, w.J.p, rows, q, w.V.p);
    auto s = nrm2 > 0 ? select(w.J.p, rows, q, true, abs2) : select(w.J.p, rows, q, false, 0);
    const int rp = (int)s.size();
    if (c.o.verbose)
      fprintf(stderr, "[vsie round] L->R k=%d core %ldx%d ||A||^2 %.6e kept %d s[0] %.6e s[last] %.6e\n", k,
              (long)rows, q, nrm2, rp, s[0].first, s.back().first);
    std::vector<int> sel(rp);
    std::vector<double> inv(rp), sv(rp);
    for (int j = 0; j < rp; ++j) {
      sel[j] = s[j].second;
      sv[j] = s[j].first;
      inv[j] = s[j].first > 0 ? 1.0 / s[j].first : 0.0;
    }
    upload_idx(c, sel);
    upload_scales(inv);
    nxt.alloc(rows * rp);
    launch_gather_cols(w.J.p, rows, rows, c.ws.idx.p, w.norms.p, rp, nxt.p, rows, false, c.st);  // U_r
    std::swap(core[k], nxt);
    upload_scales(sv);
    w.Vr.ensure((int64_t)q * rp);
    launch_gather_cols(w.V.p, q, q, c.ws.idx.p, w.norms.p, rp, w.Vr.p, q, false, c.st);  // V_r S_r
    const int64_t ncols = (int64_t)n[k + 1] * rk[k + 2];
    nxt.alloc(rp * ncols);
    zgemm1(c, kC, kN, rp, ncols, q, w.Vr.p, q, core[k + 1].p, q, nxt.p, rp);  // S_r V_r^H core_{k+1}
    std::swap(core[k + 1], nxt);
    rk[k + 1] = rp;
    sync(c);
  }
  r[0] = rk[1];
  r[1] = rk[2];
  r[2] = rk[3];
}

}  // namespace

int tt_round(vsie_coupling_s* h, double tol) {
  VSIE_REQUIRE(h->has_cores, VSIE_ERR_STATE, "handle has no TT cores");
  VSIE_REQUIRE(h->comm == nullptr, VSIE_ERR_STATE,
               "round of a multi-process handle: round the full cores before sharding");
  VSIE_REQUIRE(tol >= 0 && tol < 1, VSIE_ERR_ARG, "tol must be in [0, 1)");
  vsie_build_opts o{};
  Ctx c{h, o, nullptr, {}, tol, tol / std::sqrt(3.0), 0};
  VSIE_CHECK_CUDA(cudaDeviceSynchronize());
  VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{c.st};
  const int n[4] = {h->grid.n[0], h->grid.n[1], h->grid.n[2], (int)h->m};
  // round all three chi into new buffers first: the handle keeps its cores (and captured
  // graphs) untouched if any factorisation throws
  DevBuf<cplx> rounded[3][4];
  int rr[3][3];
  for (int chi = 0; chi < 3; ++chi) {
    int r[3] = {h->ranks[chi][0], h->ranks[chi][1], h->ranks[chi][2]};
    DevBuf<cplx>* core = rounded[chi];
    // assemble the full cores (G3 / G4 may be split over loopback shards) on c.st (a
    // non-blocking stream: plain cudaMemcpy D2D would not be ordered before its kernels)
    core[0].alloc((size_t)n[0] * r[0]);
    core[1].alloc((size_t)r[0] * n[1] * r[1]);
    core[2].alloc((size_t)r[1] * n[2] * r[2]);
    core[3].alloc((size_t)r[2] * n[3]);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(core[0].p, h->G1[chi].p, core[0].bytes(), cudaMemcpyDeviceToDevice, c.st));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(core[1].p, h->G2[chi].p, core[1].bytes(), cudaMemcpyDeviceToDevice, c.st));
    for (const Shard& s : h->shards) {
      const int64_t r2 = r[1], r3 = r[2], n3l = s.n3loc();
      if (n3l > 0)
        VSIE_CHECK_CUDA(cudaMemcpy2DAsync(core[2].p + r2 * s.i3b, r2 * n[2] * sizeof(cplx), s.G3[chi].p,
                                          r2 * n3l * sizeof(cplx), r2 * n3l * sizeof(cplx), r3,
                                          cudaMemcpyDeviceToDevice, c.st));
      if (s.mloc() > 0)
        VSIE_CHECK_CUDA(cudaMemcpyAsync(core[3].p + r3 * s.cb, s.G4[chi].p, r3 * s.mloc() * sizeof(cplx),
                                        cudaMemcpyDeviceToDevice, c.st));
    }
    round_chi(c, n, r, core);
    sync(c);
    for (int k = 0; k < 3; ++k) rr[chi][k] = r[k];
  }
  // commit: from here on the old cores are replaced; if an allocation fails the handle is
  // marked core-less (every apply then fails with VSIE_ERR_STATE) instead of half-updated
  apply_reset_graphs(h);
  try {
    for (int chi = 0; chi < 3; ++chi) {
      const cplx* dev[4] = {rounded[chi][0].p, rounded[chi][1].p, rounded[chi][2].p, rounded[chi][3].p};
      handle_set_cores_device(h, chi, rr[chi], dev);
    }
    VSIE_CHECK_CUDA(cudaDeviceSynchronize());
    handle_alloc_workspace(h);
  } catch (...) {
    h->has_cores = false;
    throw;
  }
  VSIE_CHECK_CUDA(cudaDeviceSynchronize());
  return VSIE_OK;
}

int cross_build(vsie_coupling_s* h, double tol, const vsie_build_opts& o) {
  Ctx c{h, o, nullptr, {}, tol, tol / std::sqrt(3.0), o.seed};
  VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{c.st};
  // held-out sample: uniform over [n1] x [n2] x [n3] x [m] (seeded)
  Heldout ho;
  uint64_t hs = o.seed ^ 0x5EEDull;
  const int cnt = std::max(1, o.heldout);
  ho.idx.resize(cnt);
  for (int i = 0; i < cnt; ++i)
    for (int k = 0; k < 4; ++k) ho.idx[i][k] = (int)(host_splitmix(hs) % (uint64_t)dim(h, k));
  ho.d_idx.alloc(2 * (size_t)cnt);
  ho.d_out.alloc(cnt);
  int status = VSIE_OK;
  for (int chi = 0; chi < 3; ++chi) {
    const int s = cross_chi(c, chi, ho);
    if (s != VSIE_OK) status = s;
  }
  h->entries_evaluated = c.n_eval;
  h->build_entry_s = c.t_entry;
  h->build_factor_s = c.t_factor;
  h->build_maxvol_s = c.t_maxvol;
  return status;
}

}  // namespace vsie
