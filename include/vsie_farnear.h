/*
 * vsie_farnear.h — C ABI of the far-near conductor block of the hybrid VSIE
 * (arXiv 2206.12409, PAPER.md = P:<line>).
 *
 * What the library computes:
 *   Z_cc^fn in C^{m_n x m_f}, the off-diagonal block of the conductor Galerkin
 *   matrix Z_cc between the m_n RWG functions of the "near" conductors (rows,
 *   testing) and the m_f RWG functions of the "far" conductors (columns, basis)
 *   (Eq. 11), compressed by adaptive cross approximation
 *       U V^* = ACA(Z_cc^fn)                                   (Eq. 12)
 *   and applied as U V^* j_f and V-bar U^T j_n in every GMRES matvec of the
 *   hybrid system (Eq. 15).  The library stores W = conj(V), so that
 *   Z_cc^fn ~= U W^T and (Z_cc^fn)^T ~= W U^T.
 *
 * Conventions (binding; readings R-CC1..R-CC3):
 *  - complex values are interleaved (re, im) float64 pairs (== torch.complex128);
 *  - RWG order of each side: as vsie_coupling.h (per mesh in input order, interior
 *    edges sorted by (min vertex id, max vertex id), T+ = the smaller triangle id);
 *  - entry Z[m, n] = scale * sum_{p=1..6} sum_{s=1..6} J^near_{m,p} . (G(r_p - r_s) J^far_{n,s})
 *    with the interior 3-point rule on both triangles of both RWGs and
 *    J_{+,q} = (l/6)(r_{+,q} - p+), J_{-,q} = (l/6)(p- - r_{-,q})  (36 pair interactions),
 *    G = (I + grad grad / k0^2) exp(-i k0 R) / (4 pi R);
 *  - ACA: partially pivoted (oracle/farnear.py aca() states every step): start row 0;
 *    residual row, column pivot = argmax |.| (smallest index on ties), residual column,
 *    next row = argmax |u_k| over rows not yet used; Frobenius norm of the approximant
 *    updated with the cross terms; stop when ||u_k|| ||w_k|| <= tol ||U_k W_k^T||_F,
 *    at max_rank, or when every row is used;
 *  - U: device complex128 m_n x rank, W: m_f x rank, column-major (ld = m_n, m_f).
 *
 * Ownership / errors / threading: as vsie_coupling.h (status codes VSIE_*; the
 * handle owns its device memory; caller pointers are read during the call or the
 * stream-ordered operation only; vsie_last_error_message() describes failures).
 */
#ifndef VSIE_FARNEAR_H_
#define VSIE_FARNEAR_H_

#include "vsie_coupling.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vsie_farnear_s* vsie_farnear_t;

typedef struct {
  int32_t max_rank;            /* ACA rank cap (steps), default 2048 (clamped to min(m_n, m_f)) */
  double scale_re, scale_im;   /* global prefactor of every entry, default 1 + 0i                 */
  int32_t device;              /* CUDA device ordinal, -1 = current                               */
  int32_t verbose;
} vsie_farnear_opts;

typedef struct {
  int64_t m_near, m_far;
  int32_t rank;
  int32_t stop;                /* 0 tolerance met, 1 max_rank reached, 2 every row used          */
  double est_err;              /* ||u_k|| ||w_k|| / ||U W^T||_F at the last step (ACA estimate) */
  double frob;                 /* ||U W^T||_F (the ACA recursion)                                */
  double min_distance;         /* smallest near-far quadrature node distance (m)                 */
  double max_edge;             /* longest triangle edge of either side (m)                       */
  double k0;
  double build_s;              /* wall seconds of vsie_farnear_build                             */
  int64_t entries_evaluated;   /* (m_f + m_n) per ACA step                                       */
  int64_t factor_bytes;        /* 16 rank (m_n + m_f)                                           */
  int64_t apply_calls;
} vsie_farnear_info;

void vsie_farnear_opts_default(vsie_farnear_opts* opts);

/* ACA of Z_cc^fn on the device: one cooperative kernel runs every ACA step
 * (residual row and column on the entry kernel, pivot searches, the norm recursion).
 * near / far: host triangle meshes (read during the call only).  tol > 0: relative ACA
 * tolerance (P:287 uses 1e-3).  Errors: VSIE_ERR_ARG (NULL, tol <= 0, freq <= 0),
 * VSIE_ERR_GEOMETRY (bad mesh, or a near and a far quadrature node closer than the longest
 * triangle edge of either side: the non-singular rule, reading R-CC3), VSIE_ERR_CUDA / NOMEM.  Returns
 * VSIE_WARN_NOT_CONVERGED (valid handle) when the ACA stopped at max_rank before tol. */
int32_t vsie_farnear_build(const vsie_mesh* near_meshes, int32_t n_near, const vsie_mesh* far_meshes,
                           int32_t n_far, double freq_hz, double tol, const vsie_farnear_opts* opts,
                           vsie_farnear_t* out);

/* Exact quadrature entries of Z_cc^fn: idx = device int64 [count][2] (near row, far col),
 * out = device complex128 [count].  Out-of-range indices: VSIE_ERR_ARG is not checked on
 * device; the caller keeps 0 <= row < m_n, 0 <= col < m_f. */
int32_t vsie_farnear_entries(vsie_farnear_t h, const int64_t* idx, int64_t count, void* out, void* stream);

/* Low-rank apply (device buffers, column-major, nrhs >= 1, stream-ordered):
 *  OP_N: x = j_f [m_f x nrhs] -> y = U (W^T x)        [m_n x nrhs]   (Z^fn j_f)
 *  OP_T: x = j_n [m_n x nrhs] -> y = W (U^T x)        [m_f x nrhs]   (V-bar U^T j_n, Eq. 15)
 *  OP_C: x = j_n [m_n x nrhs] -> y = conj(W) (U^H x)  [m_f x nrhs]   ((Z^fn)^H j_n) */
int32_t vsie_farnear_apply(vsie_farnear_t h, const void* x, void* y, int32_t op, int32_t nrhs, void* stream);

/* Both off-diagonal products of one GMRES matvec (Eq. 15), single RHS, two launches:
 * y_near = U W^T x_far and y_far = W U^T x_near. */
int32_t vsie_farnear_apply_pair(vsie_farnear_t h, const void* x_far, void* y_near, const void* x_near,
                                void* y_far, void* stream);

/* Copy the factors and the pivots to host (any pointer may be NULL):
 * U_host [m_n x rank], W_host [m_f x rank] complex128 column-major; rows / cols int32 [rank]:
 * the ACA pivots (i_k, j_k) in step order.  Synchronous. */
int32_t vsie_farnear_export(vsie_farnear_t h, void* U_host, void* W_host, int32_t* rows, int32_t* cols);

int32_t vsie_farnear_get_info(vsie_farnear_t h, vsie_farnear_info* out);

void vsie_farnear_destroy(vsie_farnear_t h);

#ifdef __cplusplus
}
#endif
#endif /* VSIE_FARNEAR_H_ */
