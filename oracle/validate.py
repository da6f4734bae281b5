"""Oracle O8 — parity metrics and the held-out protocol.

SURVEY.md §8c-T (T1 scale-relative entry criterion, T2 relative L2, T3
reconstruction, T4 held-out) and §8c-P35 (compression factor = #dense / #TT
elements, as an exact reduced fraction).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def entry_parity(got, ref, tol=1e-12, floor=1e-6):
    """T1: max|d| <= tol max|z|, ||d|| <= tol ||z||, and |d_i| <= tol |z_i| for
    every i with |z_i| >= floor * max|z|.  Returns (ok, worst dict)."""
    got = np.asarray(got); ref = np.asarray(ref)
    d = np.abs(got - ref)
    a = np.abs(ref)
    zmax = a.max() if a.size else 0.0
    c1 = d.max() / zmax if a.size and zmax > 0 else 0.0
    c2 = np.linalg.norm(got - ref) / np.linalg.norm(ref) if a.size and zmax > 0 else 0.0
    big = a >= floor * zmax
    c3 = (d[big] / a[big]).max() if np.any(big) else 0.0
    worst = dict(max_rel_to_max=float(c1), l2_rel=float(c2), elementwise_rel=float(c3))
    return (c1 <= tol and c2 <= tol and c3 <= tol), worst


def rel_l2(got, ref):
    ref = np.asarray(ref)
    nrm = np.linalg.norm(ref)
    return float(np.linalg.norm(np.asarray(got) - ref) / (nrm if nrm > 0 else 1.0))


def compression_factor(n, m, ranks_per_chi):
    """(3 n_v m) / sum |cores| as an exact Fraction."""
    nv = n[0] * n[1] * n[2]
    dense = 3 * nv * m
    tt = 0
    for (r1, r2, r3) in ranks_per_chi:
        tt += n[0] * r1 + r1 * n[1] * r2 + r2 * n[2] * r3 + r3 * m
    return Fraction(dense, tt)
