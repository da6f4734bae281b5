"""Oracle O5 — TT matvecs in the paper's order, plus dense TT expansion.

TT of one chi-tensor (Eq. 14):
  Z~chi[i1,i2,i3,n] = sum_{a1,a2,a3} G1[i1,a1] G2[a1,i2,a2] G3[a2,i3,a3] G4[a3,n]

Cores are held as 3-D arrays (r_{k-1}, n_k, r_k) with r0 = r4 = 1; their flat
column-major order (numpy order='F') is the C-ABI layout of §8c-L16.

Forward: y4 = G4 x; Y3 = G3 y4; Y2 = G2 Y3; y = G1 Y2, per chi, and
[y^1; y^2; y^3] stacked component-major.
Transpose: z = sum_chi ((u^chi)^T Z~chi)^T, evaluated G1 first.
Conjugate transpose (§8c-L14): Z^H u = conj(Z^T conj(u)).
"""
from __future__ import annotations

import numpy as np


def dims_of(cores):
    return tuple(c.shape[1] for c in cores)


def ranks_of(cores):
    return tuple(c.shape[2] for c in cores[:3])


def forward_one(cores, x):
    """y = Z~ x for one chi; x in C^m -> y in C^{n1 n2 n3} (i1 fastest)."""
    G1, G2, G3, G4 = cores
    y4 = G4[:, :, 0] @ x                                  # P:213  r3
    Y3 = np.einsum("bkc,c->bk", G3, y4)                   # P:214  r2 x n3
    Y2 = np.einsum("ajb,bk->ajk", G2, Y3)                 # P:215  r1 x n2 x n3
    Y = np.einsum("ia,ajk->ijk", G1[0], Y2)               # P:216  n1 x n2 x n3
    return Y.reshape(-1, order="F")


def transpose_one(cores, u):
    """z = Z~^T u for one chi; u in C^{n1 n2 n3} -> z in C^m."""
    G1, G2, G3, G4 = cores
    n1, n2, n3 = dims_of(cores)[:3]
    U = np.asarray(u).reshape((n1, n2, n3), order="F")
    W1 = np.einsum("ia,ijk->ajk", G1[0], U)               # P:231  Y G1
    W2 = np.einsum("ajb,ajk->bk", G2, W1)                 # P:232  Y G2
    z3 = np.einsum("bkc,bk->c", G3, W2)                   # P:233  y G3
    return G4[:, :, 0].T @ z3                             # P:234  y G4


def apply(tts, x, op="N"):
    """Z~ applied to x (op 'N'), Z~^T (op 'T') or Z~^H (op 'C').

    tts: list of q = 3 core lists; x: vector or [len, nrhs] (column-wise, §8c-A)."""
    x = np.asarray(x)
    if x.ndim == 2:
        return np.stack([apply(tts, x[:, j], op) for j in range(x.shape[1])], axis=1)
    if op == "N":
        return np.concatenate([forward_one(c, x) for c in tts])
    if op == "T":
        nv = int(np.prod(dims_of(tts[0])[:3]))
        z = np.zeros(dims_of(tts[0])[3], dtype=np.complex128)
        for chi, c in enumerate(tts):                     # Eq. 18: sum over chi
            z = z + transpose_one(c, x[chi * nv:(chi + 1) * nv])
        return z
    if op == "C":
        return np.conj(apply(tts, np.conj(x), "T"))
    raise ValueError(op)


def full(cores):
    """Dense 4-D tensor n1 x n2 x n3 x m of one TT (Eq. 9)."""
    G1, G2, G3, G4 = cores
    T = np.einsum("bkc,cn->bkn", G3, G4[:, :, 0])          # r2 x n3 x m
    T = np.einsum("ajb,bkn->ajkn", G2, T)                   # r1 x n2 x n3 x m
    return np.einsum("ia,ajkn->ijkn", G1[0], T)


def full_matrix(tts):
    """Dense Z~ in C^{3 n_v x m}, rows chi-major then i1 fastest (§8c-L12)."""
    blocks = []
    for c in tts:
        T = full(c)
        blocks.append(T.reshape(-1, T.shape[3], order="F"))
    return np.concatenate(blocks)


def tensor_of(Z, n, chi):
    """The 4-D chi-tensor n1 x n2 x n3 x m of a dense Z (reshape of P:109)."""
    nv = n[0] * n[1] * n[2]
    return Z[chi * nv:(chi + 1) * nv].reshape((n[0], n[1], n[2], Z.shape[1]), order="F")


def eval_at(cores, idx):
    """TT entries at an [N, 4] index list: chain product (Eq. 9, §8a-A12)."""
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 4)
    G1, G2, G3, G4 = cores
    v = G1[0][idx[:, 0], :]                                   # [N, r1]
    v = np.einsum("na,anb->nb", v, G2[:, idx[:, 1], :])
    v = np.einsum("nb,bnc->nc", v, G3[:, idx[:, 2], :])
    return np.einsum("nc,cn->n", v, G4[:, idx[:, 3], 0])


def core_elements(tts):
    return sum(int(c.size) for cores in tts for c in cores)
