/*
 * vsie_hybrid.h — C ABI of the GMRES consumer of the hybrid VSIE system
 * (arXiv 2206.12409, PAPER.md = P:<line>).
 *
 * What the library computes:
 *   the operator of the hybrid-VSIE system, Eq. 15, with unknowns
 *   x = [j_f (m_f); j_n (m_n); j_b (3 n_v)] stored contiguously (device complex128):
 *
 *     y_f = Z_cc^ff j_f + V-bar U^T j_n + (Z_cb^f)^T j_b
 *     y_n = U V^* j_f   + Z_cc^nn j_n   + (Z_cb^n)^T j_b
 *     y_b = Z_cb^f j_f  + Z_cb^n j_n    + d_b .* j_b
 *
 *   (plain transposes as Eq. 15 writes them; the lower-right 2 x 2 is Z^pFFT of P:165-167),
 *   and restarted GMRES on it ("an iterative solver, like GMRES, should be used";
 *   tolerance 1e-5, restart 50).  Blocks come from the handles of this library:
 *     Z_cc^ff  vsie_farfar_t on the far meshes,
 *     U V^*    vsie_farnear_t (near rows, far columns),
 *     Z_cc^nn  vsie_farfar_t on the near meshes (the same EFIE Galerkin machinery),
 *     Z_cb^f   vsie_coupling_t on the far meshes (the TT-compressed coupling, Eq. 14),
 *     Z_cb^n   vsie_coupling_t on the near meshes: the near coupling by the same TT machinery
 *              (the paper projects it with pFFT, P:165-172 -- DESIGN.md reading R-G1),
 *     Z_bb     its local part only, a diagonal d_b (the PWC test of M_eps_r, Eq. 2: h1 h2 h3
 *              eps_r per unknown); the nonlocal FFT-based M_chi N part is out of scope (R-G1).
 *   With no near domain (fn, nn, cb_near all NULL) m_n = 0 and the system is Eq. 4 with the
 *   far conductors only.
 *
 * GMRES (oracle/gmres.py states every step): x0 = 0; Arnoldi with classical Gram-Schmidt
 * and one full reorthogonalisation (CGS2, reading R-G2); Givens rotations on the host;
 * relative residual estimate |g_{j+1}| / ||b||; stop at <= tol or max_iter matvecs; restart
 * from x with r = b - A x.  Device: the Krylov basis V [N x (restart + 1)], the matvec, the
 * projections V^H w (fixed-order block partial sums), the updates w -= V h with the norm of
 * the result in the same pass, and x += V y.  Host: the (restart + 1) x restart Hessenberg
 * least-squares problem.
 *
 * Ownership / errors / threading: the hybrid handle references (does not own) the block
 * handles, which must outlive it and must be single-process (world 1); d_b is copied.  Status
 * codes VSIE_* as vsie_coupling.h; vsie_last_error_message() describes failures.  Calls on
 * one handle must not run concurrently (shared workspaces).
 */
#ifndef VSIE_HYBRID_H_
#define VSIE_HYBRID_H_

#include "vsie_coupling.h"
#include "vsie_farfar.h"
#include "vsie_farnear.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vsie_hybrid_s* vsie_hybrid_t;

typedef struct {
  int64_t m_far, m_near, n_body;  /* block sizes; n_body = 3 n_v                              */
  int64_t n;                      /* m_far + m_near + n_body                                  */
  int64_t matvecs;                /* vsie_hybrid_matvec / GMRES products so far               */
} vsie_hybrid_info;

typedef struct {
  int32_t iterations;             /* matvecs of the Arnoldi steps (the paper's GMRES count)  */
  int32_t restarts;               /* completed cycles                                        */
  int32_t converged;              /* 1: relative residual estimate <= tol                     */
  double rel_residual;            /* |g_{j+1}| / ||b|| at exit                               */
  double seconds;                 /* wall time of the solve                                  */
  double matvec_seconds;          /* device time of the matvecs (CUDA events)                */
} vsie_gmres_info;

/* Create the operator from built blocks.  ff, cb_far: required; fn, nn, cb_near: all set or
 * all NULL.  Sizes must agree: ff.m = fn.m_far = cb_far.m; nn.m = fn.m_near = cb_near.m;
 * cb_far and cb_near on the same voxel grid; every handle on the current device, world 1.
 * d_body: device complex128 [3 n_v] (copied).  Errors: VSIE_ERR_ARG (NULL / size mismatch /
 * multi-process handle), VSIE_ERR_CUDA / NOMEM. */
int32_t vsie_hybrid_create(vsie_farfar_t ff, vsie_farnear_t fn, vsie_farfar_t nn, vsie_coupling_t cb_far,
                           vsie_coupling_t cb_near, const void* d_body, vsie_hybrid_t* out);

/* y = A x (Eq. 15), x / y device complex128 [n] (distinct buffers), stream-ordered on
 * `stream` (NULL = default stream). */
int32_t vsie_hybrid_matvec(vsie_hybrid_t h, const void* x, void* y, void* stream);

/* Solve A x = b by restarted GMRES(restart) from x0 = 0.  b, x: device complex128 [n].
 * history: host double [max_iter] receiving the relative residual estimate after every
 * iteration, or NULL.  Synchronous (the host runs the Givens least squares; one small
 * device-to-host copy per iteration).  restart >= 1, max_iter >= 1, tol > 0, else
 * VSIE_ERR_ARG.  Returns VSIE_WARN_NOT_CONVERGED (x holds the last iterate) when max_iter
 * was reached above tol. */
int32_t vsie_hybrid_gmres(vsie_hybrid_t h, const void* b, void* x, int32_t restart, int32_t max_iter, double tol,
                          double* history, vsie_gmres_info* info, void* stream);

int32_t vsie_hybrid_get_info(vsie_hybrid_t h, vsie_hybrid_info* out);

void vsie_hybrid_destroy(vsie_hybrid_t h);

#ifdef __cplusplus
}
#endif
#endif /* VSIE_HYBRID_H_ */
