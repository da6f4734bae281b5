"""Oracle (test infrastructure; shares no code with the GPU path) — the dense far-far conductor
block Z_cc^ff of the hybrid VSIE ("Z_cc^ff ... the Galerkin
matrices that model the interactions between the m_f far ... surface discretization elements",
Eq. 11 / 15; the EFIE of Eq. 1 discretised with RWG functions).

Entry (readings R-FF1..R-FF3 of DESIGN.md): the Galerkin EFIE in mixed-potential form -- the
grad grad / k0^2 part of the dyad moved onto the divergences of the RWG test and basis
functions by integration by parts (their normal components vanish on boundary edges):

    Z[m, n] = int_Tm int_Tn [ f_m(r) . f_n(r') - div f_m div' f_n / k0^2 ] g(|r - r'|) dS' dS,

with f = s (l / 2A)(r - p), div f = s l / A on T+ (s = +1) and T- (s = -1).  Per triangle pair
(T_a of m, T_b of n) this is  s_a s_b l_m l_n / (4 A_a A_b) * K_ab,

    K_ab = sum_q (A_a / 3) int_{T_b} [ (r_q - p_a) . (r' - p_b) - 4 / k0^2 ] g(|r_q - r'|) dS'

(r_q: the interior 3-point rule on T_a).  The inner integral:
  * regular pair (|c_a - c_b| >= 2 max(L_a, L_b), c the centroids, L the longest edges): the same
    3-point rule on T_b;
  * near pair (including self and edge-adjacent pairs): g = 1/(4 pi R) + g_s with the bounded
    g_s = (exp(-i k0 R) - 1) / (4 pi R) (g_s(0) = -i k0 / (4 pi)); the 1/R part through the
    closed-form potentials I0 = int_T 1/R dS', I1 = int_T (r' - r)/R dS' of a flat triangle
    (tri_potentials), the g_s part by the 3-point rule; and K symmetrised, K_ab <- (K_ab + K_ba)/2.
The matrix is symmetric by definition: Z[m, n] is evaluated with the row the larger index.
"""
from __future__ import annotations

import numpy as np

from .geometry import TRI_BARY, rwg_edges


def rwg_triangle_tables(meshes):
    """Per RWG (canonical order, meshes concatenated): triangle vertices Vp, Vm [m, 3, 3], free
    vertices pp, pm [m, 3], length l [m]."""
    Vp, Vm, pp, pm, ln = [], [], [], [], []
    for xyz, tri in meshes:
        xyz = np.asarray(xyz, dtype=np.float64)
        tri = np.asarray(tri, dtype=np.int64)
        r = rwg_edges(xyz, tri)
        Vp.append(xyz[tri[r["tp"]]])
        Vm.append(xyz[tri[r["tm"]]])
        pp.append(xyz[r["pp"]])
        pm.append(xyz[r["pm"]])
        ln.append(r["length"])
    return dict(Vp=np.concatenate(Vp), Vm=np.concatenate(Vm), pp=np.concatenate(pp), pm=np.concatenate(pm),
                l=np.concatenate(ln))


def tri_area(V):
    return 0.5 * np.linalg.norm(np.cross(V[..., 1, :] - V[..., 0, :], V[..., 2, :] - V[..., 0, :]), axis=-1)


def longest_edge(V):
    return np.max(np.stack([np.linalg.norm(V[..., (e + 1) % 3, :] - V[..., e, :], axis=-1) for e in range(3)]),
                  axis=0)


def tri_potentials(V, r):
    """Closed-form I0 = int_T 1/|r - r'| dS' and I1 = int_T (r' - r)/|r - r'| dS' over the flat
    triangle V [3, 3] at points r [N, 3] (or batched: V [B, 3, 3], r [B, N, 3]) -- the potential
    integrals of a flat triangle: the plane height h, the in-plane projection rho, per edge i the
    unit tangent l_i (counter-clockwise about the normal), the outward normal u_i = l_i x n, the
    signed distance P0_i from rho to the edge line, the end-point abscissae l-_i, l+_i and
    distances R-_i, R+_i:
      I0 = sum_i [ P0_i ln((R+ + l+)/(R- + l-)) - |h| (atan(P0 l+ / (R0^2 + |h| R+)) - atan(P0 l- / (R0^2 + |h| R-))) ]
      int_T (rho' - rho)/R = 1/2 sum_i u_i [ R0_i^2 ln((R+ + l+)/(R- + l-)) + l+ R+ - l- R- ],
      I1 = int (rho' - rho)/R - h n I0,   R0_i^2 = P0_i^2 + h^2.
    Edge terms whose log coefficient vanishes (R0_i = 0: rho on the edge line) are dropped (the
    limit of P0 ln P0^2 is 0)."""
    V = np.asarray(V, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    single = V.ndim == 2
    if single:
        V, r = V[None], np.atleast_2d(r)[None]
    nrm = np.cross(V[:, 1] - V[:, 0], V[:, 2] - V[:, 0])
    n = nrm / np.linalg.norm(nrm, axis=-1, keepdims=True)                 # [B, 3]
    h = np.einsum("bqc,bc->bq", r - V[:, None, 0], n)                     # [B, Q]
    rho = r - h[..., None] * n[:, None, :]
    ah = np.abs(h)
    I0 = np.zeros(h.shape)
    Irho = np.zeros(r.shape)
    for i in range(3):
        a, b = V[:, i], V[:, (i + 1) % 3]
        el = np.linalg.norm(b - a, axis=-1, keepdims=True)
        lt = (b - a) / el
        u = np.cross(lt, n)
        lp = np.einsum("bqc,bc->bq", b[:, None] - rho, lt)
        lm = np.einsum("bqc,bc->bq", a[:, None] - rho, lt)
        P0 = np.einsum("bqc,bc->bq", a[:, None] - rho, u)
        R02 = P0 * P0 + h * h
        Rp = np.sqrt(R02 + lp * lp)
        Rm = np.sqrt(R02 + lm * lm)
        ok = R02 > (1e-14 * el) ** 2
        with np.errstate(divide="ignore", invalid="ignore"):
            lg = np.where(ok, np.log((Rp + lp) / (Rm + lm)), 0.0)
            at = np.where(ok, np.arctan(P0 * lp / (R02 + ah * Rp)) - np.arctan(P0 * lm / (R02 + ah * Rm)), 0.0)
        I0 += P0 * lg - ah * at
        Irho += 0.5 * (R02 * lg + lp * Rp - lm * Rm)[..., None] * u[:, None, :]
    I1 = Irho - (h * I0)[..., None] * n[:, None, :]
    return (I0[0], I1[0]) if single else (I0, I1)


def _nodes(V):
    return np.einsum("qj,...jc->...qc", TRI_BARY, V)


def _gs(R, k0):
    """(exp(-i k0 R) - 1) / (4 pi R), bounded; -i k0 / (4 pi) at R = 0."""
    R = np.asarray(R, dtype=np.float64)
    out = np.full(R.shape, -1j * k0 / (4 * np.pi), dtype=np.complex128)
    nz = R > 0
    Rn = R[nz]
    out[nz] = (np.cos(k0 * Rn) - 1.0 - 1j * np.sin(k0 * Rn)) / (4 * np.pi * Rn)
    return out


def k_regular(Va, pa, Vb, pb, k0):
    """K_ab by the 3 x 3 rule (arrays [..., 3, 3] / [..., 3])."""
    ra, rb = _nodes(Va), _nodes(Vb)
    Aa, Ab = tri_area(Va), tri_area(Vb)
    da = ra - pa[..., None, :]                       # [..., 3q, 3]
    db = rb - pb[..., None, :]                       # [..., 3s, 3]
    R = np.linalg.norm(ra[..., :, None, :] - rb[..., None, :, :], axis=-1)
    f = np.einsum("...qc,...sc->...qs", da, db) - 4.0 / k0 ** 2
    g = np.exp(-1j * k0 * R) / (4 * np.pi * R)
    return (Aa / 3) * (Ab / 3) * np.sum(f * g, axis=(-2, -1))


def k_near_oneway(Va, pa, Vb, pb, k0):
    """sum_q (A_a/3) int_{T_b} [...] g dS' with singularity subtraction (one pair [3, 3] / [3],
    or a batch [B, 3, 3] / [B, 3])."""
    Va, pa, Vb, pb = (np.asarray(x, dtype=np.float64) for x in (Va, pa, Vb, pb))
    single = Va.ndim == 2
    if single:
        Va, pa, Vb, pb = Va[None], pa[None], Vb[None], pb[None]
    ra, rb = _nodes(Va), _nodes(Vb)                                       # [B, 3, 3]
    Aa, Ab = tri_area(Va), tri_area(Vb)
    I0, I1 = tri_potentials(Vb, ra)
    da = ra - pa[:, None, :]
    sing = (np.einsum("bqc,bqc->bq", da, I1 + (ra - pb[:, None, :]) * I0[..., None]) - 4.0 / k0 ** 2 * I0) / (4 * np.pi)
    R = np.linalg.norm(ra[:, :, None, :] - rb[:, None, :, :], axis=-1)
    f = np.einsum("bqc,bsc->bqs", da, rb - pb[:, None, :]) - 4.0 / k0 ** 2
    smooth = (Ab / 3)[:, None] * np.sum(f * _gs(R, k0), axis=2)
    out = (Aa / 3) * np.sum(sing + smooth, axis=1)
    return out[0] if single else out


def is_near(Va, Vb):
    ca, cb = Va.mean(axis=-2), Vb.mean(axis=-2)
    d2 = np.sum((ca - cb) ** 2, axis=-1)
    L = np.maximum(longest_edge(Va), longest_edge(Vb))
    return d2 < (2.0 * L) ** 2


def entries_ff(T, k0, rows, cols, scale=1.0 + 0.0j):
    """Z^ff[rows[i], cols[i]] (symmetric: evaluated at (max, min))."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    m = np.maximum(rows, cols)
    n = np.minimum(rows, cols)
    out = np.zeros(len(m), dtype=np.complex128)
    for sa, Va_all, pa_all in ((1.0, T["Vp"], T["pp"]), (-1.0, T["Vm"], T["pm"])):
        for sb, Vb_all, pb_all in ((1.0, T["Vp"], T["pp"]), (-1.0, T["Vm"], T["pm"])):
            Va, pa, Vb, pb = Va_all[m], pa_all[m], Vb_all[n], pb_all[n]
            coef = sa * sb * T["l"][m] * T["l"][n] / (4 * tri_area(Va) * tri_area(Vb))
            with np.errstate(divide="ignore", invalid="ignore"):   # self pairs: replaced below
                K = k_regular(Va, pa, Vb, pb, k0)
            near = np.flatnonzero(is_near(Va, Vb))
            if near.size:
                K[near] = 0.5 * (k_near_oneway(Va[near], pa[near], Vb[near], pb[near], k0)
                                 + k_near_oneway(Vb[near], pb[near], Va[near], pa[near], k0))
            out += coef * K
    return scale * out


def dense_ff(T, k0, scale=1.0 + 0.0j):
    m = len(T["l"])
    r, c = np.tril_indices(m)
    vals = entries_ff(T, k0, r, c, scale)
    Z = np.zeros((m, m), dtype=np.complex128)
    Z[r, c] = vals
    Z[c, r] = vals
    return Z
