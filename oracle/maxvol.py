"""Oracle O6 — maxvol.

Not in the paper's text; named by BASELINE.json's north star ("maxvol on small
pivot matrices") and standard inside the cited TT-cross [oseledets2010tt]
(P:126).  Heuristic: the oracle implements the algorithm step by step and is
pinned by its invariants (P21-P23), not by pivot equality.

Input: A in C^{n x r}, n >= r, full column rank; tau = 0.05; it_max = 100 r.
 1. initial pivots = first r pivot rows of LU with partial pivoting
    (per column the row of max |.|, ties to the smallest row);
 2. B = A A[I,:]^{-1};
 3. loop: (i*, j*) = argmax |B_ij| (ties: smallest i, then j); stop if
    |B_i*j*| <= 1 + tau; else I[j*] = i*,
    B <- B - B[:, j*] (B[i*, :] - e_j*^T) / B[i*, j*].
Returns (I, B, n_swaps).  B is the interpolation matrix (B[I,:] = identity).
"""
from __future__ import annotations

import numpy as np


def lu_pivots(A):
    """Row pivots of Gaussian elimination with partial pivoting (first r)."""
    W = np.array(A, dtype=np.complex128, copy=True)
    n, r = W.shape
    perm = np.arange(n)
    for j in range(r):
        col = np.abs(W[j:, j])
        p = j + int(np.argmax(col))          # argmax returns the first max
        if p != j:
            W[[j, p], :] = W[[p, j], :]
            perm[[j, p]] = perm[[p, j]]
        if W[j, j] != 0:
            f = W[j + 1:, j] / W[j, j]
            W[j + 1:, j:] -= np.outer(f, W[j, j:])
    return perm[:r].copy()


def maxvol(A, tau=0.05, it_max=None):
    A = np.asarray(A, dtype=np.complex128)
    n, r = A.shape
    if n < r:
        raise ValueError("maxvol needs n >= r")
    if it_max is None:
        it_max = 100 * r
    I = lu_pivots(A)
    B = np.linalg.solve(A[I, :].T, A.T).T
    swaps = 0
    for _ in range(it_max):
        absB = np.abs(B)
        flat = int(np.argmax(absB))          # row-major first max: smallest i, then j
        i, j = divmod(flat, r)
        if absB[i, j] <= 1.0 + tau:
            break
        I[j] = i
        bij = B[i, j]
        row = B[i, :].copy()
        row[j] -= 1.0
        B -= np.outer(B[:, j], row) / bij
        swaps += 1
    return I, B, swaps
