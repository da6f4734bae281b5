"""Oracle O2/O3 — Z_bc entries by the plain quadrature definition, and dense Z.

Definition (PAPER.md P:106 coupling matrix, Eq. 3 dyad,
P:90 PWC testing, P:78 RWG basis; quadrature per §8c-L7):

  Z[rho, n] = scale * sum_{p=1..8} w_p sum_{s=1..6} [ G(r_p - r_s) J_s ]_chi

  row rho = chi * n_v + i1 + n1 (i2 + n2 i3)   (§8c-L12)
  col n   = RWG id in canonical order           (§8c-L10)

No approximation beyond the fixed quadrature; 48 pair interactions per entry.

PWL testing (q = 12 unknowns per voxel; "linear terms"; SURVEY §8f NEXT-2;
DESIGN.md reading R-PWL): the 12 test functions of a voxel are chi x {1, (x-c_x)/h_x,
(y-c_y)/h_y, (z-c_z)/h_z}.  `moment` l = 0 is the PWC block above; l = 1, 2, 3 multiply
every node weight w_p by the linear function at the node, (r_p - c)_l / h_l.  With one
node per voxel (ng = 1, the paper's far-block rule) the linear blocks vanish
identically, which is the "neglected" contribution of P:381.
"""
from __future__ import annotations

from dataclasses import dataclass
import math

import numpy as np

from . import geometry, greens

C0 = 299_792_458.0


@dataclass
class Problem:
    n: tuple
    h: tuple
    origin: tuple
    k0: float
    rs: np.ndarray      # [m, 6, 3] source nodes
    js: np.ndarray      # [m, 6, 3] real moment vectors
    offs: np.ndarray    # [8, 3] voxel node offsets
    wts: np.ndarray     # [8] voxel node weights
    scale: complex = 1.0 + 0.0j
    moment: int = 0     # PWL test moment (0 = PWC; 1, 2, 3 = linear in x, y, z)

    @property
    def n_v(self):
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def m(self):
        return self.rs.shape[0]

    @property
    def shape(self):
        return (3 * self.n_v, self.m)


def make_problem(n, h, origin, meshes, freq, scale=1.0 + 0.0j, ng=2, bary=None, moment=0, quad_rule=0):
    """k0 = 2 pi f / c0 (§8c-L19); sources from geometry.mesh_sources.

    moment l in 1..3: node weights w_p (r_p - c)_l / h_l (PWL test function, module header).
    quad_rule 1: the paper's far-block rule, "1 volume and 1 surface integration point" for
    Z_bc^f: ng = 1 (voxel centre, weight h1 h2 h3) and the triangle centroid
    (geometry.TRI_CENTROID, weight A); 0 keeps ng / bary (default 2 x 2 x 2 x 3-point)."""
    if moment not in (0, 1, 2, 3):
        raise ValueError("moment must be 0 (PWC) or 1..3 (linear in x, y, z)")
    if quad_rule not in (0, 1):
        raise ValueError("quad_rule must be 0 (2x2x2 x 3-point) or 1 (1 x 1, P:287)")
    if quad_rule == 1:
        ng, bary = 1, geometry.TRI_CENTROID
    rs, js = geometry.mesh_sources(meshes, geometry.TRI_BARY if bary is None else bary)
    offs, wts = geometry.gauss_legendre_offsets(h, ng)
    if moment:
        wts = wts * (offs[:, moment - 1] / h[moment - 1])
    return Problem(tuple(n), tuple(h), tuple(origin), 2.0 * math.pi * freq / C0, rs, js, offs, wts,
                   complex(scale), moment)


def problem_from_config(cfg, **kw):
    return make_problem(cfg.n, cfg.h, cfg.origin, cfg.meshes(), cfg.freq, **kw)


def field_vectors(prob: Problem, voxels, cols, chunk=8192):
    """E[b, :] = scale * sum_p w_p sum_s G(r_p - r_s) J_s for pairs (voxels[b], cols[b]).

    Returns [B, 3] complex: all three chi components of the tested field."""
    voxels = np.asarray(voxels, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    out = np.empty((len(voxels), 3), dtype=np.complex128)
    i1, i2, i3 = geometry.voxel_index(voxels, prob.n)
    cen = np.stack([prob.origin[0] + i1 * prob.h[0], prob.origin[1] + i2 * prob.h[1],
                    prob.origin[2] + i3 * prob.h[2]], axis=1)
    for s in range(0, len(voxels), chunk):
        c = cen[s:s + chunk]
        P = c[:, None, :] + prob.offs[None]                      # [B,8,3]
        rs = prob.rs[cols[s:s + chunk]]                          # [B,6,3]
        js = prob.js[cols[s:s + chunk]]
        R = P[:, :, None, :] - rs[:, None, :, :]                 # [B,8,6,3]
        GJ = greens.dyad_apply(R, js[:, None, :, :], prob.k0)    # [B,8,6,3]
        out[s:s + chunk] = prob.scale * np.einsum("p,bpsc->bc", prob.wts, GJ)
    return out


def entries(prob: Problem, rows, cols):
    """Z[rows[b], cols[b]] for explicit (row, col) lists (the black box of P:126)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if rows.size == 0:
        return np.zeros(0, dtype=np.complex128)
    chi = rows // prob.n_v
    v = rows % prob.n_v
    E = field_vectors(prob, v, cols)
    return E[np.arange(len(rows)), chi]


def tensor_entries(prob: Problem, chi: int, idx):
    """A_chi(i1, i2, i3, n) for an [N, 4] index array (the 4-D tensor of P:109-111)."""
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 4)
    v = idx[:, 0] + prob.n[0] * (idx[:, 1] + prob.n[1] * idx[:, 2])
    return entries(prob, chi * prob.n_v + v, idx[:, 3])


def dense(prob: Problem, chunk_vox=64):
    """Full Z in C^{3 n_v x m} (only for tiny configs, §8c-L23)."""
    nv, m = prob.n_v, prob.m
    Z = np.empty((3 * nv, m), dtype=np.complex128)
    cols = np.arange(m)
    for v0 in range(0, nv, chunk_vox):
        vs = np.arange(v0, min(nv, v0 + chunk_vox))
        V = np.repeat(vs, m)
        Cc = np.tile(cols, len(vs))
        E = field_vectors(prob, V, Cc).reshape(len(vs), m, 3)
        for chi in range(3):
            Z[chi * nv + vs, :] = E[:, :, chi]
    return Z
