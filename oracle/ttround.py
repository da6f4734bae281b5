"""Oracle O8 — TT rounding (recompression) of a chi-TT.  TEST INFRASTRUCTURE ONLY:
imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.

SURVEY §8(f) NEXT-1.  The paper notes that cross "might overestimate the TT-ranks"
(Discussion) and builds its TT from "a sequence of SVDs on the
unfolding matrices".  Rounding is the TT-SVD of a tensor already in TT format
(algorithm of the cited [Oseledets 2011], "TT-rounding", restated here):

  1. right-to-left orthogonalisation, k = d .. 2:
       unfold G_k as r_{k-1} x (n_k r_k);  G_k^T = Q R  (QR, Q column-orthonormal)
       G_k     <- Q^T                       (rows orthonormal)
       G_{k-1} <- G_{k-1} x_3 R^T           (carry into the left neighbour)
     after this ||A||_F = ||G_1||_F.
  2. left-to-right truncation with delta = tol / sqrt(d - 1) * ||A||_F, k = 1 .. d-1:
       unfold G_k as (r_{k-1} n_k) x r_k;  G_k = U S V^H  (SVD)
       r'_k = smallest r with ||S[r:]|| <= delta             (trunc_rank, as TT-SVD)
       G_k     <- U[:, :r']
       G_{k+1} <- (S V^H)[:r', :] x_1 G_{k+1}

  Guarantee (same theorem as TT-SVD): ||round(A) - A||_F <= tol ||A||_F, and the ranks
  are the TT-SVD ranks of A at that tolerance (up to ties at the threshold).

Cores are 3-D arrays (r_{k-1}, n_k, r_k) as in oracle/ttmv.py; d = 4 for a chi-TT.
"""
from __future__ import annotations

import numpy as np

from .ttsvd import trunc_rank


def _unfold_left(G):
    """(r_{k-1} n_k) x r_k unfolding (column-major, i.e. the C-ABI core layout)."""
    a, n, b = G.shape
    return G.reshape((a * n, b), order="F")


def _unfold_right(G):
    """r_{k-1} x (n_k r_k) unfolding."""
    a, n, b = G.shape
    return G.reshape((a, n * b), order="F")


def orthogonalize_rl(cores):
    """Step 1: right-to-left orthogonalisation; returns new cores (same tensor)."""
    G = [np.array(c, dtype=np.complex128) for c in cores]
    d = len(G)
    for k in range(d - 1, 0, -1):
        a, n, b = G[k].shape
        Q, R = np.linalg.qr(_unfold_right(G[k]).T)          # (n b) x a' , a' x a
        ap = Q.shape[1]
        G[k] = Q.T.reshape((ap, n, b), order="F")
        p, m, _ = G[k - 1].shape
        G[k - 1] = (_unfold_left(G[k - 1]) @ R.T).reshape((p, m, ap), order="F")
    return G


def tt_round(cores, tol):
    """TT rounding of one TT (list of d cores) to relative Frobenius accuracy tol."""
    G = orthogonalize_rl(cores)
    d = len(G)
    nrm = np.linalg.norm(G[0])
    delta = tol / np.sqrt(d - 1) * nrm
    for k in range(d - 1):
        a, n, b = G[k].shape
        U, S, Vh = np.linalg.svd(_unfold_left(G[k]), full_matrices=False)
        r = trunc_rank(S, delta) if nrm > 0.0 else 1
        G[k] = U[:, :r].reshape((a, n, r), order="F")
        carry = S[:r, None] * Vh[:r, :]                     # r x b
        a2, n2, b2 = G[k + 1].shape
        G[k + 1] = (carry @ _unfold_right(G[k + 1])).reshape((r, n2, b2), order="F")
    return G


def _gram_step(M, Ga, Gb):
    """M'[c, d] = sum_{a, b, i} M[a, b] Ga[a, i, c] conj(Gb[b, i, d]) (two pairwise
    contractions: the single 5-index einsum would loop over all indices at once)."""
    T = np.tensordot(M, Ga, axes=([0], [0]))                # (b, i, c)
    return np.tensordot(T, np.conj(Gb), axes=([0, 1], [0, 1]))  # (c, d)


def tt_norm(cores):
    """||A||_F of a TT by contracting the Gram chain (no dense expansion)."""
    M = np.ones((1, 1), dtype=np.complex128)
    for G in cores:
        M = _gram_step(M, G, G)
    return float(np.sqrt(abs(M[0, 0].real)))


def tt_inner(cores_a, cores_b):
    """<A, B> = sum A conj(B) of two TTs of equal dims."""
    M = np.ones((1, 1), dtype=np.complex128)
    for Ga, Gb in zip(cores_a, cores_b):
        M = _gram_step(M, Ga, Gb)
    return complex(M[0, 0])


def tt_sum(cores_a, cores_b, beta=1.0):
    """TT of A + beta B: block cores [A1 B1], diag(A_k, B_k), [A_d; beta B_d]."""
    d = len(cores_a)
    out = []
    for k, (Ga, Gb) in enumerate(zip(cores_a, cores_b)):
        a1, n, b1 = Ga.shape
        a2, _, b2 = Gb.shape
        if k == 0:
            out.append(np.concatenate([Ga, Gb], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([Ga, beta * Gb], axis=0))
        else:
            G = np.zeros((a1 + a2, n, b1 + b2), dtype=np.complex128)
            G[:a1, :, :b1] = Ga
            G[a1:, :, b1:] = Gb
            out.append(G)
    return out


def tt_diff_norm(cores_a, cores_b):
    """||A - B||_F: the TT of A - B orthogonalised right-to-left (QR, backward stable),
    then ||core_1||_F.  (The Gram identity |A|^2 + |B|^2 - 2 Re<A, B> would lose half
    the digits to cancellation when A and B are close.)"""
    return float(np.linalg.norm(orthogonalize_rl(tt_sum(cores_a, cores_b, -1.0))[0]))
