"""Oracle O1 — voxel quadrature nodes and RWG source tables.

P:78  "Coils are modeled with a triangular tessellation and the unknown j_c is
       approximated with the Rao-Wilton-Glisson (RWG) basis functions".
P:90  uniform voxelized domain n1 x n2 x n3 = n_v; PWC basis, q = 3.
P:106 Z_cb in C^{q n_v x m}, Petrov-Galerkin (PWC voxel testing, RWG basis).

Readings: L7 quadrature (2x2x2 Gauss per voxel, interior
3-point rule per triangle), L8 voxel coordinates, L10 RWG order/sign, L11
m = #RWG (interior edges).
"""
from __future__ import annotations

import numpy as np

# interior degree-2 triangle rule: barycentric rows, weights A/3 each (§8c-L7)
TRI_BARY = np.array([[2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0],
                     [1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0],
                     [1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0]])


# one point per triangle, the centroid with the whole triangle's weight: the paper's surface
# rule for the far coupling block Z_bc^f ("1 volume and 1 surface integration point")
TRI_CENTROID = np.array([[1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0]])


class GeometryError(ValueError):
    pass


def voxel_centres(n, h, origin):
    """Centre of voxel (i1,i2,i3) = origin + (i1 h1, i2 h2, i3 h3) (§8c-L8).

    Returned in the row order of Z: v = i1 + n1 (i2 + n2 i3) (§8c-L12)."""
    i1, i2, i3 = voxel_index(np.arange(n[0] * n[1] * n[2]), n)
    return np.stack([origin[0] + i1 * h[0], origin[1] + i2 * h[1], origin[2] + i3 * h[2]], axis=1)


def voxel_index(v, n):
    """Decode the column-major voxel id v = i1 + n1 (i2 + n2 i3) (§8c-L12)."""
    v = np.asarray(v, dtype=np.int64)
    return v % n[0], (v // n[0]) % n[1], v // (n[0] * n[1])


def gauss_legendre_offsets(h, ng: int = 2):
    """Tensor Gauss-Legendre rule on a voxel of size h centred at 0.

    Returns (offsets [ng^3, 3], weights [ng^3]).  ng = 2 gives c +- h/(2 sqrt 3)
    with weights h1 h2 h3 / 8 (§8c-E).  Node order: sigma1 fastest."""
    x, w = np.polynomial.legendre.leggauss(ng)
    offs, wts = [], []
    for c in range(ng):
        for b in range(ng):
            for a in range(ng):
                offs.append([x[a] * h[0] / 2, x[b] * h[1] / 2, x[c] * h[2] / 2])
                wts.append(w[a] * w[b] * w[c] * h[0] * h[1] * h[2] / 8.0)
    return np.array(offs), np.array(wts)


def rwg_edges(xyz, tri):
    """Interior edges of one triangle mesh -> RWG functions (§8c-L10).

    Returns a dict of int64/float arrays, one entry per RWG, in canonical order
    (interior edges sorted by (min vertex id, max vertex id)):
      a, b       shared-edge vertex ids (a < b)
      tp, tm     T+ (adjacent triangle with the smaller id) and T-
      pp, pm     vertex of T+ / T- opposite the shared edge
      length     |v_a - v_b|
    Raises GeometryError for degenerate triangles or non-manifold edges."""
    xyz = np.asarray(xyz, dtype=np.float64)
    tri = np.asarray(tri, dtype=np.int64)
    e1 = xyz[tri[:, 1]] - xyz[tri[:, 0]]
    e2 = xyz[tri[:, 2]] - xyz[tri[:, 0]]
    area = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
    if np.any(area <= 0.0) or np.any(tri < 0) or np.any(tri >= len(xyz)):
        raise GeometryError("degenerate triangle or vertex id out of range")
    edges = {}
    for t in range(len(tri)):
        for k in range(3):
            a, b = tri[t, (k + 1) % 3], tri[t, (k + 2) % 3]
            key = (min(a, b), max(a, b))
            edges.setdefault(key, []).append((t, tri[t, k]))
    out = {k: [] for k in ("a", "b", "tp", "tm", "pp", "pm", "length")}
    for key in sorted(edges):
        adj = edges[key]
        if len(adj) > 2:
            raise GeometryError(f"edge {key} shared by {len(adj)} triangles")
        if len(adj) < 2:
            continue  # boundary edge: no RWG
        adj = sorted(adj)
        (tp, pp), (tm, pm) = adj
        out["a"].append(key[0]); out["b"].append(key[1])
        out["tp"].append(tp); out["tm"].append(tm)
        out["pp"].append(pp); out["pm"].append(pm)
        out["length"].append(np.linalg.norm(xyz[key[0]] - xyz[key[1]]))
    return {k: np.array(v) for k, v in out.items()}


def source_table(xyz, tri, rwg, bary=TRI_BARY):
    """Per RWG: source nodes r_s [m, 2*nq, 3] and real moment vectors J_s.

    On T+ with vertices (v0, v1, v2) (stored order): r_{+,q} = sum_j bary[q,j] v_j,
    J_{+,q} = (l/6)(r_{+,q} - p+); on T-: J_{-,q} = (l/6)(p- - r_{-,q}).
    This is f_n = +-(l/2A)(r - p) times the rule weight A/3 (§8c-E); for a
    general rule with weights w_q (sum 1) pass bary and the factor becomes
    l/2 * w_q... here the 3-point rule with w_q = 1/3 gives l/6."""
    xyz = np.asarray(xyz, dtype=np.float64)
    tri = np.asarray(tri, dtype=np.int64)
    nq = bary.shape[0]
    wq = 1.0 / nq
    m = len(rwg["length"])
    rs = np.empty((m, 2 * nq, 3))
    js = np.empty((m, 2 * nq, 3))
    vp = xyz[tri[rwg["tp"]]]  # [m,3,3]
    vm = xyz[tri[rwg["tm"]]]
    rp = np.einsum("qj,mjc->mqc", bary, vp)
    rm = np.einsum("qj,mjc->mqc", bary, vm)
    l = rwg["length"][:, None, None]
    rs[:, :nq] = rp
    rs[:, nq:] = rm
    js[:, :nq] = (l / 2.0) * wq * (rp - xyz[rwg["pp"]][:, None, :])
    js[:, nq:] = (l / 2.0) * wq * (xyz[rwg["pm"]][:, None, :] - rm)
    return rs, js


def mesh_sources(meshes, bary=TRI_BARY):
    """Concatenate RWG source tables of several surfaces in input order (§8c-L10)."""
    rs_all, js_all = [], []
    for xyz, tri in meshes:
        rwg = rwg_edges(xyz, tri)
        rs, js = source_table(xyz, tri, rwg, bary)
        rs_all.append(rs)
        js_all.append(js)
    return np.concatenate(rs_all), np.concatenate(js_all)


def node_box_distance(n, h, origin, rs, ng=2):
    """Distance from the source nodes to the axis-aligned bounding box of all
    voxel quadrature nodes: a lower bound on the minimum voxel-node /
    source-node distance, used for the non-singularity check (DESIGN.md
    reading R-L18: build fails when this is < 10 max(h))."""
    offs, _ = gauss_legendre_offsets(h, ng)
    lo = np.array([origin[a] + offs[:, a].min() for a in range(3)])
    hi = np.array([origin[a] + (n[a] - 1) * h[a] + offs[:, a].max() for a in range(3)])
    src = np.asarray(rs).reshape(-1, 3)
    d = np.linalg.norm(np.maximum(0.0, np.maximum(lo - src, src - hi)), axis=1)
    return float(d.min())
