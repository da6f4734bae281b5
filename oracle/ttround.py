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


def tt_norm(cores):
    """||A||_F of a TT by contracting the Gram chain (no dense expansion)."""
    M = np.ones((1, 1), dtype=np.complex128)
    for G in cores:
        # M'[b, b'] = sum_{a, a', i} M[a, a'] G[a, i, b] conj(G[a', i, b'])
        M = np.einsum("ab,aic,bid->cd", M, G, np.conj(G))
    return float(np.sqrt(abs(M[0, 0].real)))


def tt_inner(cores_a, cores_b):
    """<A, B> = sum A conj(B) of two TTs of equal dims."""
    M = np.ones((1, 1), dtype=np.complex128)
    for Ga, Gb in zip(cores_a, cores_b):
        M = np.einsum("ab,aic,bid->cd", M, Ga, np.conj(Gb))
    return complex(M[0, 0])


def tt_diff_norm(cores_a, cores_b):
    """||A - B||_F from Gram chains: sqrt(|A|^2 + |B|^2 - 2 Re<A, B>)."""
    na2 = tt_norm(cores_a) ** 2
    nb2 = tt_norm(cores_b) ** 2
    v = na2 + nb2 - 2.0 * tt_inner(cores_a, cores_b).real
    return float(np.sqrt(max(v, 0.0)))
