"""Oracle O4 — TT-SVD ("a sequence of SVDs on the unfolding
matrices"; algorithm of the cited [Oseledets2011] as restated in SURVEY §8c-S).

Used only as a reference (ranks on the tiny config, P19) — the method itself
builds the TT by cross, never by TT-SVD.
"""
from __future__ import annotations

import numpy as np


def trunc_rank(s, delta_abs):
    """Smallest r >= 1 with ||s[r:]||_2 <= delta_abs."""
    tail = np.sqrt(np.cumsum((s[::-1] ** 2))[::-1])  # tail[r] = ||s[r:]||
    tail = np.append(tail, 0.0)
    for r in range(1, len(s) + 1):
        if tail[r] <= delta_abs:
            return r
    return len(s)


def tt_svd(A, tol):
    """TT of a d-way array A with ||A - TT||_F <= tol ||A||_F.

    Per-unfolding threshold delta = tol / sqrt(d-1) * ||A||_F (theorem of
    Oseledets 2011)."""
    A = np.asarray(A, dtype=np.complex128)
    dims = A.shape
    d = len(dims)
    nrm = np.linalg.norm(A)
    delta = tol / np.sqrt(d - 1) * nrm
    cores = []
    r_prev = 1
    C = A.reshape((dims[0], -1), order="F")
    for k in range(d - 1):
        C = C.reshape((r_prev * dims[k], -1), order="F")
        if nrm == 0.0:
            U = np.zeros((C.shape[0], 1), dtype=np.complex128)
            S = np.zeros(1)
            Vh = np.zeros((1, C.shape[1]), dtype=np.complex128)
            r = 1
        else:
            U, S, Vh = np.linalg.svd(C, full_matrices=False)
            r = trunc_rank(S, delta)
        cores.append(U[:, :r].reshape((r_prev, dims[k], r), order="F"))
        C = S[:r, None] * Vh[:r, :]
        r_prev = r
    cores.append(C.reshape((r_prev, dims[d - 1], 1), order="F"))
    return cores
