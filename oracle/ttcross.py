"""Oracle O7 — DMRG two-site TT-cross with full-supercore SVD.

PAPER.md P:126 (TT-cross calls an index->value function as a black box),
P:128 (needs only a fraction of the entries), P:174-182 / Eq. 14 (TT-cross
"based on the adaptive density matrix renormalization group", q independent
4-D tensors, cores G1, G2, G3, G4).  The paper names the method only; the
concrete parameters are the readings of SURVEY.md §8c-X / L17, restated here
step by step:

 index sets nested: I_{<=k} subset I_{<=k-1} x [n_k], J_{>k} subset [n_{k+1}] x J_{>k+1}
 supercore M_k[(a, i_k), (i_{k+1}, b)] = A(I_{<=k-1}[a], i_k, i_{k+1}, J_{>k+1}[b]),
   row a + r_{k-1} i_k, col i_{k+1} + n_{k+1} b.
 0. r_k = 1; J sets from one seeded index (passed in), nested by construction.
 1. L->R, k = 1..d-1: SVD M_k = U S V^H; r = min{rho: ||s[rho:]|| <= tol/sqrt(d-1) ||s||};
    L = U[:, :r]; P = maxvol(L); I_{<=k} from P; core k = L L[P]^{-1};
    at k = d-1 also G_d = M_{d-1}[P, :].
 2. R->L, k = d-1..1: same M_k; R = (V^H)[:r, :]^T (so that M ~ X R^T, DESIGN.md
    reading R1); Q = maxvol(R); J_{>k} from Q; core k+1 = (R R[Q]^{-1})^T;
    at k = 1 also G_1 = M_1[:, Q].
 3. after each full sweep: held-out relative error e on a seeded sample
    (passed in) excluding indices lying on a pivot cross; stop when every rank
    moved by at most max(1, 5%) over the sweep and e <= 10 tol (the
    acceptance bound of §8c-L15; reading R2); at most max_sweeps;
    the TT with the smallest e is returned, flagged not-converged if e > 10 tol.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .maxvol import maxvol
from .ttsvd import trunc_rank
from . import ttmv


@dataclass
class CrossResult:
    cores: list
    ranks: tuple
    sweeps: int
    heldout_err: float
    converged: bool
    entries_evaluated: int
    I: dict = field(default_factory=dict)
    J: dict = field(default_factory=dict)
    history: list = field(default_factory=list)


def _supercore_index(I_left, n_k, n_k1, J_right):
    rl, rr = len(I_left), len(J_right)
    rows = []
    for b in range(rr):
        for i1 in range(n_k1):
            for i0 in range(n_k):
                for a in range(rl):
                    rows.append(I_left[a] + (i0, i1) + J_right[b])
    return np.array(rows, dtype=np.int64), (rl * n_k, n_k1 * rr)


def on_cross(idx, I, J, d):
    """Mask of indices lying on a pivot cross: prefix in I_{<=k} and suffix in J_{>k}."""
    mask = np.zeros(len(idx), dtype=bool)
    for k in range(1, d):
        Ik, Jk = set(I.get(k, [])), set(J.get(k, []))
        for t, row in enumerate(idx):
            if tuple(int(v) for v in row[:k]) in Ik and tuple(int(v) for v in row[k:]) in Jk:
                mask[t] = True
    return mask


def tt_cross(entry_fn, dims, tol, start_index, heldout_idx, rmax=2048, max_sweeps=8, tau=0.05):
    """TT-cross of the tensor whose entries entry_fn([N, d] int64) -> [N] complex returns."""
    d = len(dims)
    if d != 4:
        raise ValueError("the Z_bc tensors are 4-D (P:111); d must be 4")
    start_index = tuple(int(v) for v in start_index)
    I = {0: [()]}
    J = {d: [()]}
    for k in range(d - 1, 0, -1):
        J[k] = [start_index[k:]]
    ranks = [1] * (d + 1)
    cores = [None] * d
    n_eval = 0
    delta = tol / np.sqrt(d - 1)
    hv = entry_fn(np.asarray(heldout_idx, dtype=np.int64))
    n_eval += len(hv)
    best = None
    prev_ranks = None
    history = []
    sweep = 0
    for sweep in range(1, max_sweeps + 1):
        for k in range(1, d):                                     # L -> R
            idx, shape = _supercore_index(I[k - 1], dims[k - 1], dims[k], J[k + 1])
            M = entry_fn(idx).reshape(shape, order="F")
            n_eval += idx.shape[0]
            U, S, Vh = np.linalg.svd(M, full_matrices=False)
            r = trunc_rank(S, delta * np.linalg.norm(S)) if S[0] > 0 else 1
            r = max(1, min(r, rmax, *M.shape))
            P, B, _ = maxvol(U[:, :r], tau=tau)
            rl = ranks[k - 1]
            I[k] = [I[k - 1][p % rl] + (int(p // rl),) for p in P]
            cores[k - 1] = B.reshape((rl, dims[k - 1], r), order="F")
            ranks[k] = r
            if k == d - 1:
                cores[d - 1] = M[P, :].reshape((r, dims[d - 1], 1), order="F")
        for k in range(d - 1, 0, -1):                             # R -> L
            idx, shape = _supercore_index(I[k - 1], dims[k - 1], dims[k], J[k + 1])
            M = entry_fn(idx).reshape(shape, order="F")
            n_eval += idx.shape[0]
            U, S, Vh = np.linalg.svd(M, full_matrices=False)
            r = trunc_rank(S, delta * np.linalg.norm(S)) if S[0] > 0 else 1
            r = max(1, min(r, rmax, *M.shape))
            R = Vh[:r, :].T
            Q, B, _ = maxvol(R, tau=tau)
            nk1 = dims[k]
            J[k] = [(int(q % nk1),) + J[k + 1][q // nk1] for q in Q]
            cores[k] = B.T.reshape((r, nk1, ranks[k + 1]), order="F")
            ranks[k] = r
            if k == 1:
                cores[0] = M[:, Q].reshape((1, dims[0], r), order="F")
        mask = ~on_cross(heldout_idx, I, J, d)
        approx = ttmv.eval_at(cores, np.asarray(heldout_idx)[mask])
        ref = hv[mask]
        nrm = np.linalg.norm(ref)
        e = np.linalg.norm(approx - ref) / nrm if nrm > 0 else np.linalg.norm(approx - ref)
        cur = tuple(ranks[1:d])
        history.append((cur, e))
        if best is None or e < best[1]:
            best = ([c.copy() for c in cores], e, cur)
        if prev_ranks is not None and e <= 10 * tol and all(
                abs(a - b) <= max(1, b // 20) for a, b in zip(prev_ranks, cur)):
            break
        prev_ranks = cur
    cores_b, e_b, r_b = best
    return CrossResult(cores_b, r_b, sweep, e_b, e_b <= 10 * tol, n_eval,
                       {k: list(v) for k, v in I.items()}, {k: list(v) for k, v in J.items()}, history)
