/*
 * vsie_farfar.h — C ABI of the dense far-far conductor block of the hybrid VSIE
 * (arXiv 2206.12409, PAPER.md = P:<line>).
 *
 * What the library computes:
 *   Z_cc^ff in C^{m_f x m_f}, the Galerkin EFIE matrix of the m_f RWG functions of the
 *   "far" conductors (Eq. 11; the EFIE of Eq. 1, with RWG basis and
 *   testing), stored dense (the paper applies it "with standard matrix
 *   multiplications") and applied in every GMRES matvec (Eq. 15, first row).
 *
 * Conventions (binding; readings R-FF1..R-FF3; oracle/farfar.py states each step):
 *  - mixed-potential form: Z[m, n] = sum over the triangle pairs (T_a of m, T_b of n) of
 *      s_a s_b l_m l_n / (4 A_a A_b) K_ab,
 *      K_ab = sum_q (A_a/3) int_{T_b} [ (r_q - p_a).(r' - p_b) - 4/k0^2 ] g(|r_q - r'|) dS',
 *    g = exp(-i k0 R) / (4 pi R), r_q the interior 3-point rule, s = +1 on T+, -1 on T-;
 *  - regular pairs (centroid distance >= 2 x the longer longest edge): the 3-point rule on T_b;
 *    near pairs (self, adjacent, close): the 1/(4 pi R) part by the closed-form potentials of a
 *    flat triangle, the bounded rest by the 3-point rule, K symmetrised (K_ab + K_ba) / 2;
 *  - Z is symmetric by definition (evaluated with the larger index as the row);
 *  - storage: the lower triangle in 128 x 128 tiles (tile (I, J), I >= J, column-major inside,
 *    zero-padded at the ragged end): 16 * 128^2 * nb (nb + 1) / 2 bytes, nb = ceil(m_f / 128),
 *    half of the dense matrix; the apply reads every stored tile once for both Z_IJ x_J and
 *    Z_IJ^T x_I;
 *  - RWG order, complex layout, scale, ownership, errors, threading: as vsie_coupling.h.
 */
#ifndef VSIE_FARFAR_H_
#define VSIE_FARFAR_H_

#include "vsie_coupling.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vsie_farfar_s* vsie_farfar_t;

typedef struct {
  int64_t m;                 /* far RWG functions                                      */
  int32_t tile;              /* 128                                                    */
  int64_t tiles;             /* nb (nb + 1) / 2 stored tiles                           */
  int64_t matrix_bytes;      /* device bytes of the stored lower triangle              */
  int64_t near_pairs;        /* triangle pairs evaluated with the singular rule (build) */
  double build_s;            /* wall seconds of vsie_farfar_build                      */
  double k0;
  int64_t apply_calls;
} vsie_farfar_info;

/* Assemble Z_cc^ff on device (one kernel over the stored tiles).  meshes: the far surfaces
 * (host arrays, read during the call).  scale_re + i scale_im multiplies every entry (pass
 * 1, 0 for the plain matrix).  device: CUDA ordinal, -1 = current.  Errors:
 * VSIE_ERR_ARG (NULL, n_meshes < 1, freq <= 0, non-finite scale), VSIE_ERR_GEOMETRY (bad mesh),
 * VSIE_ERR_NOMEM (the tiles do not fit), VSIE_ERR_CUDA. */
int32_t vsie_farfar_build(const vsie_mesh* meshes, int32_t n_meshes, double freq_hz, double scale_re,
                          double scale_im, int32_t device, vsie_farfar_t* out);

/* Entries through the entry kernel (not the stored tiles): idx = device int64 [count][2]
 * (row, col), out = device complex128 [count]; 0 <= row, col < m (unchecked on device). */
int32_t vsie_farfar_entries(vsie_farfar_t h, const int64_t* idx, int64_t count, void* out, void* stream);

/* y = op(Z) x (+ y when accumulate != 0) on device, x / y complex128 [m x nrhs] column-major,
 * stream-ordered.  OP_N and OP_T are the same product (Z = Z^T); OP_C = conj(Z) x.
 * Two launches per RHS column (tile pass, fixed-order partial sum). */
int32_t vsie_farfar_apply(vsie_farfar_t h, const void* x, void* y, int32_t op, int32_t nrhs, int32_t accumulate,
                          void* stream);

/* The full dense matrix to host (m x m complex128, column-major), expanded from the tiles. */
int32_t vsie_farfar_export(vsie_farfar_t h, void* host_dense);

int32_t vsie_farfar_get_info(vsie_farfar_t h, vsie_farfar_info* out);

void vsie_farfar_destroy(vsie_farfar_t h);

#ifdef __cplusplus
}
#endif
#endif /* VSIE_FARFAR_H_ */
