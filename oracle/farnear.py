"""Oracle (test infrastructure; shares no code with the GPU path) — the far-near conductor block
Z_cc^fn of the hybrid VSIE (Eq. 11 row 2) and its ACA
compression U V^* (Eq. 12; used as U V^* and V-bar U^T in Eq. 15).

Entry (readings R-CC1 / R-CC2 of DESIGN.md): the Galerkin interaction between RWG m of the
near conductors (testing) and RWG n of the far conductors (basis), by the same non-singular
quadrature and dyadic form as Z_bc (§8c-E, §8c-L6) with the voxel test function replaced by
the RWG one -- the interior 3-point rule on both triangles of both RWGs, 6 x 6 = 36 pair
interactions per entry:

    Z[m, n] = scale * sum_{p=1..6} sum_{s=1..6} J^near_{m,p} . ( G(r^near_{m,p} - r^far_{n,s}) J^far_{n,s} )

with J_{+,q} = (l/6)(r_{+,q} - p+), J_{-,q} = (l/6)(p- - r_{-,q}) on each side and G the dyad of
oracle/greens.py.  G is symmetric and even, so Z^nf = (Z^fn)^T (reciprocity, pin
P43).  The surfaces are disjoint (non-singular rule; the singular self-terms of Z_cc^ff are
out of scope).

ACA: partially pivoted adaptive cross approximation (the "ACA method" of P:159 citing Zhao
2005), written out step by step: A ~= U W^T with W = conj(V) of the paper's U V^*, so the
transposed product of Eq. 15 row 1 is V-bar U^T = W U^T.
"""
from __future__ import annotations

import numpy as np

from . import greens


def entries_cc(rs_a, js_a, rs_b, js_b, k0, rows, cols, scale=1.0 + 0.0j):
    """Z[rows[i], cols[i]] for the RWG sets a (testing, rows) and b (basis, columns)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    ra, ja = rs_a[rows], js_a[rows]          # [N, 6, 3]
    rb, jb = rs_b[cols], js_b[cols]
    out = np.zeros(rows.shape[0], dtype=np.complex128)
    for p in range(ra.shape[1]):
        for s in range(rb.shape[1]):
            R = ra[:, p, :] - rb[:, s, :]
            gj = greens.dyad_apply(R, jb[:, s, :], k0)          # G(R) J_s
            out += np.sum(ja[:, p, :] * gj, axis=-1)              # J_p . (G J_s)
    return scale * out


def dense_cc(rs_a, js_a, rs_b, js_b, k0, scale=1.0 + 0.0j):
    ma, mb = rs_a.shape[0], rs_b.shape[0]
    r, c = np.meshgrid(np.arange(ma), np.arange(mb), indexing="ij")
    return entries_cc(rs_a, js_a, rs_b, js_b, k0, r.ravel(), c.ravel(), scale).reshape(ma, mb)


def aca(row_fn, col_fn, m, n, tol, max_rank=None, pivots=None, trace=None):
    """Partially pivoted ACA of an m x n matrix given by row_fn(i) -> A[i, :] and
    col_fn(j) -> A[:, j].  Returns (U [m, k], W [n, k]) with A ~= U W^T.

    pivots: optional [(i_k, j_k)] to replay another run's pivot sequence (near-ties of |.| on a
    rotationally symmetric geometry make the argmax order-dependent); the steps below are
    unchanged, only the two argmax choices are replaced, and when trace is a list it receives
    per step (|rrow[j_k]| / max_j |rrow|, |u_{k-1}[i_k]| / max_unused |u_{k-1}|) -- both 1 for
    a valid ACA pivot.

    Step k (rows I, columns J used so far; S_{k-1} = sum_{l<k} u_l w_l^T):
      1. residual row  rrow = A[i_k, :] - sum_l U[i_k, l] w_l
      2. j_k = argmax_j |rrow_j| (ties: smallest j); if rrow[j_k] == 0 the row is exhausted:
         mark it used and take the next row (step 6)
      3. w_k = rrow / rrow[j_k]
      4. u_k = A[:, j_k] - sum_l U[:, l] w_l[j_k]
      5. ||S_k||_F^2 = ||S_{k-1}||_F^2 + 2 Re sum_l (u_l^H u_k)(w_l^H w_k) + ||u_k||^2 ||w_k||^2;
         stop when ||u_k|| ||w_k|| <= tol ||S_k||_F
      6. i_{k+1} = argmax over unused rows of |u_k| (ties: smallest i)
    """
    if max_rank is None:
        max_rank = min(m, n)
    U = np.zeros((m, 0), dtype=np.complex128)
    W = np.zeros((n, 0), dtype=np.complex128)
    used = np.zeros(m, dtype=bool)
    norm2 = 0.0
    i = 0
    row_ratio = 1.0
    while U.shape[1] < max_rank and not used.all():
        if pivots is not None:
            if U.shape[1] >= len(pivots):
                break
            i = int(pivots[U.shape[1]][0])
            if U.shape[1] > 0:
                au = np.abs(U[:, -1]).copy()
                au[used] = -1.0
                row_ratio = abs(U[i, -1]) / au.max() if au.max() > 0 else 1.0
        rrow = np.asarray(row_fn(i), dtype=np.complex128) - U[i, :] @ W.T
        used[i] = True
        j = int(np.argmax(np.abs(rrow)))
        if pivots is not None:
            jf = int(pivots[U.shape[1]][1])
            if trace is not None:
                trace.append((abs(rrow[jf]) / abs(rrow[j]) if abs(rrow[j]) > 0 else 1.0, row_ratio))
            j = jf
        if abs(rrow[j]) == 0.0:
            cand = np.flatnonzero(~used)
            if cand.size == 0:
                break
            i = int(cand[0])
            continue
        w = rrow / rrow[j]
        u = np.asarray(col_fn(j), dtype=np.complex128) - U @ W[j, :]
        cross = 2.0 * np.real(np.sum((U.conj().T @ u) * (W.conj().T @ w)))
        nu, nw = np.linalg.norm(u), np.linalg.norm(w)
        norm2 += cross + (nu * nw) ** 2
        U = np.concatenate([U, u[:, None]], axis=1)
        W = np.concatenate([W, w[:, None]], axis=1)
        if nu * nw <= tol * np.sqrt(max(norm2, 0.0)) and pivots is None:
            break
        au = np.abs(u)
        au[used] = -1.0
        i = int(np.argmax(au))
        if au[i] < 0:
            break
    return U, W


def apply_lowrank(U, W, x, op="N"):
    """op N: y = U (W^T x) (near rows = Z^fn x_far); T: W (U^T x) (= (Z^fn)^T x_near, the V-bar
    U^T product of Eq. 15 row 1); C: conj(W) (U^H x) (= (Z^fn)^H x_near)."""
    if op == "N":
        return U @ (W.T @ x)
    if op == "T":
        return W @ (U.T @ x)
    if op == "C":
        return W.conj() @ (U.conj().T @ x)
    raise ValueError(op)
