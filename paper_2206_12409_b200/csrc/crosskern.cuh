// Device kernels of the TT-cross driver: rank-revealing
// factorisation of supercores (one-sided Jacobi SVD, randomized range finder
// sketches), maxvol (LU-initialised, rank-1 updates) and index gathers.
#pragma once

#include "common.cuh"

namespace vsie {

// complex normal (a + ib)/sqrt 2 from a counter-based generator (splitmix64 + Box-Muller)
void launch_gaussian(cplx* out, int64_t n, uint64_t seed, cudaStream_t st);

// one round of the parallel one-sided (Hestenes) Jacobi method on the columns of
// A (p x q, ld lda), accumulating the same rotations into V (q x q, ld q) if V != null.
// pairs: int2[npairs] column pairs; rotations applied counted into *rot_count.
void launch_jacobi_round(cplx* A, int64_t p, int64_t lda, cplx* V, int64_t q, const int2* pairs, int npairs,
                         double thr, double small2, unsigned* rot_count, cudaStream_t st);
// all sweeps in one cooperative launch (npairs CTAs must be co-resident; returns
// false without launching otherwise).  cnt: 3 unsigned, zeroed by the caller;
// cnt[2] = sweeps performed.
bool launch_jacobi_coop(cplx* A, int64_t p, int64_t lda, cplx* V, int64_t q, const int2* pairs, int npairs,
                        int nrounds, double thr, double small2, int max_sweeps, unsigned* cnt, cudaStream_t st);
// out[j] = ||A[:, j]||_2
void launch_col_norms(const cplx* A, int64_t p, int64_t q, int64_t lda, double* out, cudaStream_t st);
// sum |a_i|^2 (deterministic two-pass) -> *out (device)
void launch_frob2(const cplx* A, int64_t n, double* partial /*>= 1024*/, double* out, cudaStream_t st);

// dst[:, j] = scale_j * src[:, idx[j]]  (idx, scale on device; scale may be null; conj optional)
void launch_gather_cols(const cplx* src, int64_t rows, int64_t lds, const int* idx, const double* scale, int ncols,
                        cplx* dst, int64_t ldd, bool conj, cudaStream_t st);
// dst[i, :] = src[idx[i], :]   (dst nr x cols, ld nr)
void launch_gather_rows(const cplx* src, int64_t lds, const int* idx, int nr, int64_t cols, cplx* dst,
                        cudaStream_t st);
// dst (rows x cols, ld rows) = conj(src (ld lds)); conj of C (rows x cols, ld ldc) in place
void launch_copy_conj(const cplx* src, int64_t lds, int64_t rows, int64_t cols, cplx* dst, cudaStream_t st);
void launch_conj_2d(cplx* C, int64_t ldc, int64_t rows, int64_t cols, cudaStream_t st);
// dst[i, :] = src[idx[i] - r0, :] for idx[i] in [r0, r1), else 0 (row-split matrices)
void launch_gather_rows_owned(const cplx* src, int64_t lds, const int* idx, int nr, int64_t cols, int64_t r0,
                              int64_t r1, cplx* dst, cudaStream_t st);
// dst (C x R) = op(src (R x C)), op = transpose or conj-transpose
void launch_transpose(const cplx* src, int64_t R, int64_t C, cplx* dst, bool conj, cudaStream_t st);

// ---- Cholesky QR pieces (shifted CholeskyQR3 preconditioning of the Jacobi SVD)
// G[i + q i] += s for i < q
void launch_add_diag(cplx* G, int q, double s, cudaStream_t st);
// in-place upper Cholesky of the Hermitian q x q matrix G (upper triangle used):
// on exit G holds R (upper, G = R^H R), strictly lower part zeroed.  *bad set if a
// pivot was not positive.
void launch_cholesky_upper(cplx* G, int q, int* bad, cudaStream_t st);
// X = R^{-1} for upper triangular R (q x q, column-major); Rt = scratch q x q
void launch_upper_inverse(const cplx* R, int q, cplx* Rt, cplx* X, cudaStream_t st);
// sum of the real diagonal of G -> *out (device)
void launch_trace_real(const cplx* G, int q, double* out, cudaStream_t st);

// ---- blocked Householder QR (hqr.cu) ---------------------------------------------------
struct HqrWs {
  cplx* V;          // >= p x panel width
  cplx* W;          // >= panel width x n (trailing / applied columns)
  cplx* W2;         // same
  cplx* Gv;         // >= panel width^2
  double* part;     // >= hqr_part_doubles()
  cplx* zws;        // ZGEMM split-K workspace
  int64_t zws_elems;
};
int hqr_panels(int q);
int hqr_panel_width();
size_t hqr_part_doubles();
// A (p x q, ld lda, p >= q) = Q R in place (R upper, reflectors below the diagonal); tau[q];
// T: hqr_panels(q) panel factors of panel width^2 complex each
void hqr_factor(cplx* A, int64_t lda, int64_t p, int q, cplx* tau, cplx* T, const HqrWs& w, cudaStream_t st);
// C (p x n, ld ldc) <- Q C with Q from hqr_factor
void hqr_apply_q(const cplx* A, int64_t lda, int64_t p, int q, const cplx* T, cplx* C, int64_t ldc, int n,
                 const HqrWs& w, cudaStream_t st);
// R (q x q, ld q) <- upper triangle of A (zero below)
void hqr_copy_r(const cplx* A, int64_t lda, int q, cplx* R, cudaStream_t st);
// C (p x n) <- [B; 0] (B q x n, ld ldb) or the first n columns of the identity
void hqr_fill(const cplx* B, int64_t ldb, int q, int64_t p, int n, cplx* C, int64_t ldc, bool identity,
              cudaStream_t st);

// ---- maxvol -------------------------------------------------------------
struct ArgMax {
  double v;     // |value|^2
  int64_t key;  // tie-break key (smaller wins)
  int64_t i;    // row (permuted frame)
  int c;        // column
};

// LU with partial pivoting of W (n x r, ld n), in place, rows physically swapped;
// perm[i] = original row of permuted row i.  Step j: scale column j and update columns
// (j, c1) on rows > j (scale), then argmax partials of column j + 1 (argmax); j = -1: argmax
// of column 0 only.  Blocked: panels of kLuPanel columns, the trailing matrix updated per
// panel by launch_lu_trsm (U12 = L11^{-1} A12) and a ZGEMM A22 -= L21 U12.
constexpr int kLuPanel = 32;
void launch_lu_update(cplx* W, int64_t n, int r, int j, int c1, bool scale, bool argmax, ArgMax* partials, int nparts,
                      cudaStream_t st);
void launch_lu_trsm(cplx* W, int64_t n, int r, int j0, int jb, cudaStream_t st);
void launch_lu_pivot(cplx* W, int64_t n, int r, int j, int* perm, const ArgMax* partials, int nparts,
                     int* bad, cudaStream_t st);
int lu_nparts(int64_t n);
// Lr[i * r + k] = W[i + n k] for k < i (strict lower of the leading r x r), row-major
void launch_copy_lower(const cplx* W, int64_t n, int r, cplx* Lr, cudaStream_t st);
// T = inverse of the unit lower triangular matrix whose strict lower part is Lr (row-major); T column-major r x r
void launch_unit_lower_inverse(const cplx* Lr, int r, cplx* T, cudaStream_t st);
// B[0:r, 0:r] = identity (B ld n)
void launch_set_identity_top(cplx* B, int64_t n, int r, cudaStream_t st);

struct MaxvolState {
  int i_star, c_star;  // chosen element (permuted frame)
  cplx piv;            // B[i*, c*]
  int done;            // 1: converged (max |B| <= 1 + tau) or it cap
  int swaps;
  double maxabs;       // |B[i*, c*]| of the last selection
};
// argmax pass (update = false) or rank-1 update + argmax pass over B (n x r, ld n)
void launch_maxvol_update(cplx* B, int64_t n, int r, const int* perm, const cplx* rowbuf, const MaxvolState* s,
                          bool update, ArgMax* partials, int nparts, cudaStream_t st);
void launch_maxvol_select(cplx* B, int64_t n, int r, const ArgMax* partials, int nparts, double tau,
                          int* piv_pos, cplx* rowbuf, MaxvolState* s, cudaStream_t st);
// Bout[perm[i], :] = B[i, :]
void launch_scatter_rows(const cplx* B, int64_t n, int r, const int* perm, cplx* Bout, cudaStream_t st);

}  // namespace vsie
