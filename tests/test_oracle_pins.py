"""Pins of the CPU oracle against things other than itself.

Each test names the pin id (P1..P35) and what fixes it: a closed form, an
extended-precision (mpmath, 40 digits) recomputation, a textbook quadrature
fact, an invariant of the mathematics, or brute force on tiny inputs.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import synth
from gpu_common import inflate as _inflate
from oracle import entries, geometry, greens, maxvol, ttcross, ttmv, ttround, ttsvd, validate

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
K0 = 2 * np.pi * synth.configs.FREQ_7T / synth.configs.C0


# ---------------------------------------------------------------- Green's function

def test_P5_g_closed_forms():
    # k0 = 0 static limit, phase wrap at k0 R = 2 pi, k0 = 1, R = 2
    assert abs(greens.g_scalar(0.7, 0.0) - 1 / (4 * np.pi * 0.7)) < 1e-15
    R = 2 * np.pi / K0
    assert abs(greens.g_scalar(R, K0) - 1 / (4 * np.pi * R)) < 1e-15 / R
    ref = (np.cos(2.0) - 1j * np.sin(2.0)) / (8 * np.pi)
    assert abs(greens.g_scalar(2.0, 1.0) - ref) < 1e-16


def _mp_dyad(Rv, k0, dps=40):
    """(I + grad grad / k0^2) g by mpmath numerical differentiation at 40 digits."""
    with mp.workdps(dps):
        k = mp.mpf(k0)
        def g(x, y, z):
            R = mp.sqrt(x * x + y * y + z * z)
            return mp.exp(-1j * k * R) / (4 * mp.pi * R)
        X = [mp.mpf(float(c)) for c in Rv]
        D = np.empty((3, 3), dtype=complex)
        g0 = g(*X)
        for i in range(3):
            for j in range(3):
                order = [0, 0, 0]
                order[i] += 1
                order[j] += 1
                d2 = mp.diff(g, X, tuple(order))
                D[i, j] = complex((1 if i == j else 0) * g0 + d2 / (k * k))
        return D


def test_P2_dyad_closed_form_vs_mpmath_derivatives():
    rng = np.random.default_rng(2)
    for _ in range(4):
        Rv = rng.normal(size=3)
        Rv *= rng.uniform(0.1, 3.0) / np.linalg.norm(Rv)
        ref = _mp_dyad(Rv, K0)
        got = greens.dyad(Rv, K0)
        assert np.max(np.abs(got - ref)) <= 1e-14 * np.max(np.abs(ref))
        # dyad_apply is the same operator applied to a real vector
        J = rng.normal(size=3)
        assert np.max(np.abs(greens.dyad_apply(Rv, J, K0) - ref @ J)) <= 1e-14 * np.max(np.abs(ref @ J))


def test_P1_trace_identity():
    # Helmholtz: lap g = -k0^2 g  =>  tr G = 3 g + lap g / k0^2 = 2 g
    rng = np.random.default_rng(1)
    Rv = rng.normal(size=(200, 3)) * rng.uniform(0.05, 5.0, size=(200, 1))
    D = greens.dyad(Rv, K0)
    tr = np.trace(D, axis1=-2, axis2=-1)
    g = greens.g_scalar(np.linalg.norm(Rv, axis=1), K0)
    assert np.max(np.abs(tr / g - 2.0)) < 1e-14


def test_P3_symmetry_and_parity():
    rng = np.random.default_rng(3)
    Rv = rng.normal(size=(50, 3))
    D = greens.dyad(Rv, K0)
    assert np.max(np.abs(D - np.swapaxes(D, -1, -2))) <= 1e-15 * np.max(np.abs(D))
    assert np.max(np.abs(D - greens.dyad(-Rv, K0))) <= 1e-15 * np.max(np.abs(D))


def test_P4_far_field_transversality():
    rh = np.array([0.3, -0.5, 0.8]); rh /= np.linalg.norm(rh)
    devs = []
    for R in (2.0, 5.0, 20.0, 50.0):
        D = greens.dyad(R * rh, K0)
        g = greens.g_scalar(R, K0)
        far = g * (np.eye(3) - np.outer(rh, rh))
        devs.append(np.max(np.abs(D - far)) / abs(g))
    assert all(a > b for a, b in zip(devs, devs[1:]))
    assert devs[-1] < 1e-2


# ---------------------------------------------------------------- quadrature

def test_P6_gauss2_exact_to_cubics():
    h = (0.3, 0.5, 0.7)
    offs, w = geometry.gauss_legendre_offsets(h, 2)
    for p in itertools.product(range(5), repeat=3):
        if max(p) > 4:
            continue
        num = np.sum(w * np.prod(offs ** np.array(p), axis=1))
        exact = 1.0
        for a in range(3):
            k = p[a]
            exact *= 0.0 if k % 2 else 2 * (h[a] / 2) ** (k + 1) / (k + 1)
        if max(p) <= 3:
            assert abs(num - exact) < 1e-15 * max(1.0, abs(exact)) + 1e-18
        elif p.count(4) == 1 and sum(p) == 4:
            assert abs(num - exact) > 1e-6 * abs(exact)   # quartics are NOT exact


def test_P7_triangle_rule_exact_to_quadratics():
    v = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])   # reference triangle, area 1/2
    pts = geometry.TRI_BARY @ v
    for a in range(4):
        for b in range(4 - a):
            num = 0.5 / 3 * np.sum(pts[:, 0] ** a * pts[:, 1] ** b)
            exact = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
            if a + b <= 2:
                assert abs(num - exact) < 1e-15
            elif a + b == 3 and (a == 3 or b == 3):
                assert abs(num - exact) > 1e-4


def test_P8_weights():
    h = (5e-3, 4e-3, 3e-3)
    _, w = geometry.gauss_legendre_offsets(h, 2)
    assert abs(w.sum() - np.prod(h)) < 1e-15 * np.prod(h)
    assert np.allclose(w, np.prod(h) / 8, rtol=0, atol=1e-22)
    assert abs(geometry.TRI_BARY.sum(axis=1) - 1).max() < 1e-15


# ---------------------------------------------------------------- mesh / RWG

def test_P11_mesh_counts():
    for N_az, N_ax in ((24, 16), (72, 47), (88, 57), (80, 63), (100, 67), (90, 74)):
        xyz, tri = synth.cylinder_mesh(0.34, 1.2, N_az, N_ax)
        assert len(tri) == 2 * N_az * N_ax
        edges = {tuple(sorted((t[i], t[(i + 1) % 3]))) for t in tri for i in range(3)}
        assert len(edges) == N_az * (3 * N_ax + 1)
        if N_az == 24:
            r = geometry.rwg_edges(xyz, tri)
            assert len(r["a"]) == N_az * (3 * N_ax - 1) == 1128
    assert synth.get_config(3).m == 30000 and synth.get_config(4).m == 39890


def test_P9_P10_rwg_moments(prob1, cfg1):
    xyz, tri = cfg1.meshes()[0]
    rwg = geometry.rwg_edges(xyz, tri)
    rs, js = prob1.rs, prob1.js
    for n in range(0, len(rwg["a"]), 37):
        a, b = xyz[rwg["a"][n]], xyz[rwg["b"][n]]
        l = np.linalg.norm(a - b)
        pp, pm = xyz[rwg["pp"][n]], xyz[rwg["pm"][n]]
        cp = xyz[tri[rwg["tp"][n]]].mean(0)
        cm = xyz[tri[rwg["tm"][n]]].mean(0)
        # P10: sum_s J_s = (l/2)[(c+ - p+) + (p- - c-)]
        ref = 0.5 * l * ((cp - pp) + (pm - cm))
        assert np.max(np.abs(js[n].sum(0) - ref)) < 1e-14 * np.linalg.norm(ref)
        # P9: recover f_n = J_q / (A/3) at the nodes; f is linear, so extrapolate to
        # the edge midpoint and check the normal component is 1 from both sides.
        for side, (T, p, sgn) in enumerate(((rwg["tp"][n], pp, 1), (rwg["tm"][n], pm, -1))):
            V = xyz[tri[T]]
            A = 0.5 * np.linalg.norm(np.cross(V[1] - V[0], V[2] - V[0]))
            J = js[n, 3 * side:3 * side + 3]
            r = rs[n, 3 * side:3 * side + 3]
            coef = (J / (A / 3.0)) / (sgn * (r - p))               # = l/(2A) per component
            c = coef[np.abs(sgn * (r - p)) > 1e-9 * l]
            assert np.max(np.abs(c - l / (2 * A))) < 1e-12 * l / (2 * A)
            mid = 0.5 * (a + b)
            normal = np.cross(np.cross(V[1] - V[0], V[2] - V[0]), b - a)
            normal /= np.linalg.norm(normal)
            if np.dot(normal, mid - p) < 0:
                normal = -normal          # points away from p, i.e. T+ -> T- on T+
            f = sgn * l / (2 * A) * (mid - p)
            assert abs(abs(np.dot(f, normal)) - 1.0) < 1e-12


# ---------------------------------------------------------------- entries

def _mp_entry(cfg, rwg_idx, chi, vox, one_point=False):
    """P12: one entry at 40 digits, from the definitions (f_n = l/(2A)(r - p) with the
    area-weighted 3-point rule; dyad by mpmath differentiation of g).  one_point (P51): the
    paper's far-block rule of P:287, the triangle centroid with weight A and the voxel centre
    with weight h1 h2 h3."""
    xyz, tri = cfg.meshes()[0]
    rwg = geometry.rwg_edges(xyz, tri)
    a, b = rwg["a"][rwg_idx], rwg["b"][rwg_idx]
    adj = [t for t in range(len(tri)) if a in tri[t] and b in tri[t]]
    assert len(adj) == 2
    tp, tm = sorted(adj)
    mp.mp.dps = 40
    P = lambda v: [mp.mpf(float(c)) for c in v]
    va, vb = P(xyz[a]), P(xyz[b])
    l = mp.sqrt(sum((va[i] - vb[i]) ** 2 for i in range(3)))
    i1, i2, i3 = vox
    c = [mp.mpf(float(cfg.origin[0])) + i1 * mp.mpf(float(cfg.h[0])),
         mp.mpf(float(cfg.origin[1])) + i2 * mp.mpf(float(cfg.h[1])),
         mp.mpf(float(cfg.origin[2])) + i3 * mp.mpf(float(cfg.h[2]))]
    hh = [mp.mpf(float(x)) for x in cfg.h]
    k0 = 2 * mp.pi * mp.mpf(synth.configs.FREQ_7T) / mp.mpf(synth.configs.C0)
    total = mp.mpc(0)
    for sgn, T in ((1, tp), (-1, tm)):
        V = [P(xyz[v]) for v in tri[T]]
        p = [P(xyz[v]) for v in tri[T] if v not in (a, b)][0]
        e1 = [V[1][i] - V[0][i] for i in range(3)]
        e2 = [V[2][i] - V[0][i] for i in range(3)]
        cr = [e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]]
        A = mp.sqrt(sum(x * x for x in cr)) / 2
        for q in range(1 if one_point else 3):
            bary = [mp.mpf(1) / 6] * 3
            bary[q] = mp.mpf(2) / 3
            if one_point:
                bary = [mp.mpf(1) / 3] * 3
            rq = [sum(bary[j] * V[j][i] for j in range(3)) for i in range(3)]
            f = [sgn * l / (2 * A) * (rq[i] - p[i]) for i in range(3)]
            for sig in ([(0, 0, 0)] if one_point else itertools.product((-1, 1), repeat=3)):
                rp = [c[i] + sig[i] * hh[i] / (2 * mp.sqrt(3)) for i in range(3)]
                w = hh[0] * hh[1] * hh[2] / (1 if one_point else 8)
                R = [rp[i] - rq[i] for i in range(3)]
                def g(x, y, z):
                    rr = mp.sqrt(x * x + y * y + z * z)
                    return mp.exp(-1j * k0 * rr) / (4 * mp.pi * rr)
                row = []
                for j in range(3):
                    order = [0, 0, 0]
                    order[chi] += 1
                    order[j] += 1
                    row.append((g(*R) if j == chi else 0) + mp.diff(g, R, tuple(order)) / k0 ** 2)
                total += w * (A if one_point else A / 3) * sum(row[j] * f[j] for j in range(3))
    return complex(total)


@pytest.mark.slow
def test_P12_entry_extended_precision(prob1, cfg1):
    for (n, chi, vox) in ((5, 0, (0, 3, 11)), (700, 2, (6, 6, 6))):
        ref = _mp_entry(cfg1, n, chi, vox)
        v = vox[0] + cfg1.n[0] * (vox[1] + cfg1.n[1] * vox[2])
        got = entries.entries(prob1, [chi * cfg1.n_v + v], [n])[0]
        assert abs(got - ref) <= 1e-14 * abs(ref), (got, ref)


def test_P13_reciprocity(prob1, cfg1):
    """Swapped roles: sum_s sum_p J_s . G(r_s - r_p) e_chi w_p equals the entry."""
    rng = np.random.default_rng(13)
    rows = rng.integers(0, 3 * cfg1.n_v, 30)
    cols = rng.integers(0, prob1.m, 30)
    got = entries.entries(prob1, rows, cols)
    for t in range(30):
        chi, v = divmod(int(rows[t]), cfg1.n_v)
        i1, i2, i3 = geometry.voxel_index(v, cfg1.n)
        c = np.array(cfg1.origin) + np.array([i1, i2, i3]) * np.array(cfg1.h)
        acc = 0j
        for p in range(8):
            rp = c + prob1.offs[p]
            for s in range(6):
                D = greens.dyad(prob1.rs[cols[t], s] - rp, prob1.k0)   # G(r_s - r_p)
                acc += prob1.wts[p] * (prob1.js[cols[t], s] @ D)[chi]
        assert abs(acc - got[t]) <= 1e-13 * abs(got[t])


def _subdivided_rule(L):
    """3-point interior rule on the 4^L midpoint sub-triangles, as barycentrics."""
    tris = [np.eye(3)]
    for _ in range(L):
        nxt = []
        for T in tris:
            m01, m12, m20 = (T[0] + T[1]) / 2, (T[1] + T[2]) / 2, (T[2] + T[0]) / 2
            nxt += [np.array([T[0], m01, m20]), np.array([m01, T[1], m12]),
                    np.array([m20, m12, T[2]]), np.array([m01, m12, m20])]
        tris = nxt
    return np.concatenate([geometry.TRI_BARY @ T for T in tris])


def test_P14_quadrature_convergence(cfg1):
    """Refining either rule converges monotonically; the 2x2x2 / 3-point error is reported."""
    meshes = cfg1.meshes()
    row, col = [0 * cfg1.n_v + 5 + 12 * 7], [400]
    seq_v = []
    for ng in (2, 3, 4, 5):
        p = entries.make_problem(cfg1.n, cfg1.h, cfg1.origin, meshes, cfg1.freq, ng=ng, bary=_subdivided_rule(2))
        seq_v.append(entries.entries(p, row, col)[0])
    seq_t = []
    for L in (0, 1, 2, 3):
        p = entries.make_problem(cfg1.n, cfg1.h, cfg1.origin, meshes, cfg1.freq, ng=4, bary=_subdivided_rule(L))
        seq_t.append(entries.entries(p, row, col)[0])
    dv = [abs(a - b) for a, b in zip(seq_v, seq_v[1:])]
    dt = [abs(a - b) for a, b in zip(seq_t, seq_t[1:])]
    assert all(x > y for x, y in zip(dt, dt[1:])), dt
    assert dv[0] > dv[-1], dv
    assert dt[-1] < 1e-3 * abs(seq_t[-1])


def test_P15_point_dipole_limit():
    """Far away (quasi-static k0 D << 1, where the multipole remainder is O(size/D)),
    an RWG acts like a point dipole of moment sum_s J_s."""
    xyz = np.array([[0, -0.01, 0], [0, 0.01, 0], [0.015, 0, 0.002], [-0.012, 0.001, 0]], dtype=float)
    tri = np.array([[0, 1, 2], [1, 0, 3]], dtype=np.int32)
    errs = []
    for D in (0.5, 1.0, 2.0, 4.0):
        shifted = xyz + np.array([D, 0.3 * D, 0.1])
        p = entries.make_problem((1, 1, 1), (4e-3,) * 3, (0.0, 0.0, 0.0), [(shifted, tri)], 1.0e6)
        E = entries.field_vectors(p, [0], [0])[0]
        cen = p.rs[0].mean(0)
        dip = (4e-3) ** 3 * greens.dyad_apply(-cen, p.js[0].sum(0), p.k0)
        errs.append(np.max(np.abs(E - dip)) / np.max(np.abs(dip)))
    assert all(a > b for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 5e-3


def test_P16_c2_rotation_symmetry(dense1, cfg1):
    xyz, tri = cfg1.meshes()[0]
    N_az = cfg1.surfaces[0].n_az
    rwg = geometry.rwg_edges(xyz, tri)
    def vmap(v):
        k, j = divmod(int(v), N_az)
        return k * N_az + (j + N_az // 2) % N_az
    def tmap(t):
        q, s = divmod(int(t), 2)
        k, j = divmod(q, N_az)
        return 2 * (k * N_az + (j + N_az // 2) % N_az) + s
    lookup = {(int(a), int(b)): n for n, (a, b) in enumerate(zip(rwg["a"], rwg["b"]))}
    nmap, sig = [], []
    for n in range(len(rwg["a"])):
        a, b = vmap(rwg["a"][n]), vmap(rwg["b"][n])
        n2 = lookup[(min(a, b), max(a, b))]
        nmap.append(n2)
        sig.append(1.0 if tmap(rwg["tp"][n]) == rwg["tp"][n2] else -1.0)
    nmap, sig = np.array(nmap), np.array(sig)
    assert (sig < 0).sum() > 0
    n1, n2, n3 = cfg1.n
    nv = cfg1.n_v
    v = np.arange(nv)
    i1, i2, i3 = geometry.voxel_index(v, cfg1.n)
    Rv = (n1 - 1 - i1) + n1 * ((n2 - 1 - i2) + n2 * i3)
    scale = np.abs(dense1).max()
    for chi, c in ((0, -1.0), (1, -1.0), (2, 1.0)):
        Zc = dense1[chi * nv:(chi + 1) * nv]
        lhs = Zc[Rv][:, nmap]
        rhs = c * sig[None, :] * Zc
        assert np.max(np.abs(lhs - rhs)) <= 1e-13 * scale


def test_P17_golden_dense_summary(dense1, cfg1):
    with open(os.path.join(GOLDEN, "cfg1_dense_summary.json")) as f:
        g = json.load(f)
    nv = cfg1.n_v
    for chi in range(3):
        nrm = np.linalg.norm(dense1[chi * nv:(chi + 1) * nv])
        assert abs(nrm - g["fro"][chi]) <= 1e-13 * g["fro"][chi]
    W = synth.complex_gaussian(dense1.size, g["checksum_seed"]).reshape(dense1.shape)
    cs = np.sum(W * dense1)
    ref = complex(g["checksum"][0], g["checksum"][1])
    assert abs(cs - ref) <= 1e-12 * abs(ref)


# ---------------------------------------------------------------- TT-SVD

def _rand_tt(dims, ranks, seed):
    rng = np.random.default_rng(seed)
    rr = (1,) + tuple(ranks) + (1,)
    return [(rng.normal(size=(rr[k], dims[k], rr[k + 1])) + 1j * rng.normal(size=(rr[k], dims[k], rr[k + 1])))
            for k in range(len(dims))]


def test_P18_P19_ttsvd_bound_and_ranks(dense1, cfg1):
    for chi in range(3):
        A = ttmv.tensor_of(dense1, cfg1.n, chi)
        cores = ttsvd.tt_svd(A, 1e-8)
        err = np.linalg.norm(ttmv.full(cores) - A) / np.linalg.norm(A)
        assert err <= 1e-8
        r = ttmv.ranks_of(cores)
        # informational (P19): probe at 1-pt voxel rule gave (7,31,73) / z (7,30,73)
        assert 5 <= r[0] <= 9 and 25 <= r[1] <= 37 and 65 <= r[2] <= 81, r


def test_P20_ttsvd_special_cases():
    dims = (5, 6, 7, 8)
    vs = [np.random.default_rng(k).normal(size=d) + 1j for k, d in enumerate(dims)]
    A = np.einsum("i,j,k,l->ijkl", *vs)
    assert ttmv.ranks_of(ttsvd.tt_svd(A, 1e-12)) == (1, 1, 1)
    Z = np.zeros(dims, dtype=complex)
    c = ttsvd.tt_svd(Z, 1e-6)
    assert ttmv.ranks_of(c) == (1, 1, 1) and np.all(ttmv.full(c) == 0)
    i = np.arange(10)
    H = 1.0 / (i[:, None, None, None] + i[None, :, None, None] + i[None, None, :, None] + i[None, None, None, :] + 1)
    c = ttsvd.tt_svd(H, 1e-6)
    assert np.linalg.norm(ttmv.full(c) - H) <= 1e-6 * np.linalg.norm(H)
    assert max(ttmv.ranks_of(c)) <= 8


# ---------------------------------------------------------------- maxvol

def test_P21_maxvol_invariants():
    rng = np.random.default_rng(21)
    for (n, r) in ((50, 5), (200, 17), (31, 30)):
        A = rng.normal(size=(n, r)) + 1j * rng.normal(size=(n, r))
        I0 = maxvol.lu_pivots(A)
        I, B, swaps = maxvol.maxvol(A, tau=0.05)
        assert len(set(I.tolist())) == r
        assert np.max(np.abs(B[I] - np.eye(r))) < 1e-12
        assert np.max(np.abs(B)) <= 1.05 + 1e-12
        assert np.max(np.abs(B - A @ np.linalg.inv(A[I]))) < 1e-10 * max(1, np.abs(B).max())
        d0 = abs(np.linalg.det(A[I0]))
        d1 = abs(np.linalg.det(A[I]))
        assert d1 >= d0 * (1.05 ** swaps) * (1 - 1e-10)


def test_P22_maxvol_brute_force_hadamard_bound():
    rng = np.random.default_rng(22)
    for (n, r) in ((8, 2), (10, 3), (12, 4)):
        A = rng.normal(size=(n, r)) + 1j * rng.normal(size=(n, r))
        I, _, _ = maxvol.maxvol(A, tau=0.05)
        dI = abs(np.linalg.det(A[I]))
        bound = (np.sqrt(r) * 1.05) ** r
        best = max(abs(np.linalg.det(A[list(J)])) for J in itertools.combinations(range(n), r))
        assert best <= bound * dI * (1 + 1e-12)


def test_P23_maxvol_identity_top():
    rng = np.random.default_rng(23)
    r = 6
    C = rng.uniform(-0.6, 0.6, size=(30, r)) + 1j * rng.uniform(-0.6, 0.6, size=(30, r))
    A = np.vstack([np.eye(r), C])
    I, B, swaps = maxvol.maxvol(A)
    assert list(I) == list(range(r)) and swaps == 0


# ---------------------------------------------------------------- TT-cross

def _cross_on(T, tol, seed=0):
    dims = T.shape
    fn = lambda idx: T[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]]
    hi = synth.uniform_indices(dims, 300, 1000 + seed)
    st = synth.uniform_indices(dims, 1, 2000 + seed)[0]
    return ttcross.tt_cross(fn, dims, tol, st, hi)


def test_P24_cross_recovers_random_tt():
    for ranks, seed in (((2, 3, 2), 1), ((3, 5, 4), 2)):
        cores = _rand_tt((12, 12, 12, 64), ranks, seed)
        T = ttmv.full(cores)
        res = _cross_on(T, 1e-12, seed)
        assert res.ranks == ranks
        assert np.linalg.norm(ttmv.full(res.cores) - T) <= 1e-12 * np.linalg.norm(T)


def test_P25_cross_rank_one_cases():
    dims = (6, 7, 8, 9)
    C = np.full(dims, 2.5 - 1j)
    assert _cross_on(C, 1e-10).ranks == (1, 1, 1)
    vs = [np.random.default_rng(k).normal(size=d) + 0.5j for k, d in enumerate(dims)]
    S = np.einsum("i,j,k,l->ijkl", *vs)
    res = _cross_on(S, 1e-10)
    assert res.ranks == (1, 1, 1)
    assert np.linalg.norm(ttmv.full(res.cores) - S) <= 1e-12 * np.linalg.norm(S)


def test_P26_cross_cfg1_vs_dense(dense1, cfg1):
    dims = cfg1.n + (dense1.shape[1],)
    hi = synth.uniform_indices(dims, 1000, synth.SEEDS["heldout"])
    for chi in range(3):
        A = ttmv.tensor_of(dense1, cfg1.n, chi)
        fn = lambda idx: A[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]]
        st = synth.uniform_indices(dims, 1, synth.SEEDS["cross"] + chi)[0]
        res = ttcross.tt_cross(fn, dims, cfg1.tol, st, hi)
        err = np.linalg.norm(ttmv.full(res.cores) - A) / np.linalg.norm(A)
        assert err <= 10 * cfg1.tol, (chi, err, res.ranks)
        assert res.converged


# ---------------------------------------------------------------- TT matvecs

DIMS = (5, 6, 7, 9)


def _tts(seed=0, ranks=(3, 4, 5)):
    return [_rand_tt(DIMS, ranks, seed + 10 * chi) for chi in range(3)]


def test_P28_matvec_vs_dense_expansion():
    tts = _tts()
    Zt = ttmv.full_matrix(tts)
    x = synth.complex_gaussian(DIMS[3], 1)
    u = synth.complex_gaussian(3 * 5 * 6 * 7, 2)
    assert validate.rel_l2(ttmv.apply(tts, x, "N"), Zt @ x) < 1e-13
    assert validate.rel_l2(ttmv.apply(tts, u, "T"), Zt.T @ u) < 1e-13
    assert validate.rel_l2(ttmv.apply(tts, u, "C"), Zt.conj().T @ u) < 1e-13
    # element-wise: the dense expansion agrees with the chain evaluation (Eq. 9)
    idx = synth.uniform_indices(DIMS, 50, 3)
    T0 = ttmv.full(tts[0])
    assert np.allclose(ttmv.eval_at(tts[0], idx), T0[tuple(idx.T)], rtol=1e-13, atol=0)


def test_P29_adjoint_identities():
    tts = _tts(5)
    x = synth.complex_gaussian(DIMS[3], 4)
    u = synth.complex_gaussian(3 * 5 * 6 * 7, 5)
    lhs = np.sum(ttmv.apply(tts, x, "N") * u)            # bilinear, no conjugation
    rhs = np.sum(x * ttmv.apply(tts, u, "T"))
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    lhs = np.vdot(ttmv.apply(tts, x, "N"), u)
    rhs = np.vdot(x, ttmv.apply(tts, u, "C"))
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def test_P30_special_cases():
    tts = _tts(7)
    assert np.all(ttmv.apply(tts, np.zeros(DIMS[3], complex), "N") == 0)
    Zt = ttmv.full_matrix(tts)
    e = np.zeros(DIMS[3], complex); e[4] = 1
    assert np.allclose(ttmv.apply(tts, e, "N"), Zt[:, 4], rtol=1e-14, atol=1e-14 * np.abs(Zt).max())
    ones = [[np.ones((1, d, 1), complex) if k < 3 else np.ones((1, d, 1), complex) for k, d in enumerate(DIMS)]] * 3
    y = ttmv.apply(ones, np.ones(DIMS[3], complex), "N")
    assert np.all(y == DIMS[3])


def test_P31_P32_block_and_linearity():
    tts = _tts(9)
    X = synth.complex_gaussian(DIMS[3], 6, ncols=8)
    Y = ttmv.apply(tts, X, "N")
    for j in range(8):
        assert np.array_equal(Y[:, j], ttmv.apply(tts, X[:, j], "N"))
    a, b = 0.3 - 2j, 1.7 + 0.2j
    lhs = ttmv.apply(tts, a * X[:, 0] + b * X[:, 1], "N")
    rhs = a * Y[:, 0] + b * Y[:, 1]
    assert validate.rel_l2(lhs, rhs) < 1e-13


def test_P35_compression_factor_exact():
    f = validate.compression_factor((12, 12, 12), 1128, [(7, 31, 73)] * 3)
    dense = 3 * 1728 * 1128
    tt = 3 * (12 * 7 + 7 * 12 * 31 + 31 * 12 * 73 + 73 * 1128)
    assert f == Fraction(dense, tt) and isinstance(f, Fraction)


def test_T1_entry_parity_metric():
    ref = np.array([1.0, 1e-9, -2.0 + 1j, 0.0])
    ok, _ = validate.entry_parity(ref * (1 + 1e-14), ref)
    assert ok
    bad = ref.copy(); bad[2] += 1e-10
    ok, w = validate.entry_parity(bad, ref)
    assert not ok and w["elementwise_rel"] > 1e-12


# ---------------------------------------------------------------- TT rounding (§8f NEXT-1)

def test_P36_round_recovers_inflated_ranks():
    # a TT padded with redundant (linearly dependent) rank directions is the same tensor;
    # rounding at 1e-12 must return the minimal ranks and the tensor (vs dense expansion)
    for ranks, seed in (((2, 3, 2), 36), ((3, 5, 4), 37)):
        cores = _rand_tt((6, 7, 8, 20), ranks, seed)
        T = ttmv.full(cores)
        fat = _inflate(cores, 3, seed)
        assert np.linalg.norm(ttmv.full(fat) - T) <= 1e-12 * np.linalg.norm(T)
        out = ttround.tt_round(fat, 1e-12)
        assert ttmv.ranks_of(out) == ranks
        assert np.linalg.norm(ttmv.full(out) - T) <= 1e-12 * np.linalg.norm(T)


def test_P37_round_equals_ttsvd_ranks_and_bound():
    # rounding a TT is the TT-SVD of the tensor it represents (same unfoldings' singular
    # values): ranks equal TT-SVD's of the dense tensor, error within tol ||A||
    i = np.arange(9)
    H = 1.0 / (i[:, None, None, None] + i[None, :, None, None] + 2 * i[None, None, :, None]
               + 0.5 * i[None, None, None, :] + 1.0) + 0.0j
    exact = ttsvd.tt_svd(H, 1e-15)
    fat = _inflate(exact, 2, 38)
    for tol in (1e-3, 1e-6, 1e-9):
        out = ttround.tt_round(fat, tol)
        ref = ttsvd.tt_svd(H, tol)
        assert ttmv.ranks_of(out) == ttmv.ranks_of(ref), (tol, ttmv.ranks_of(out), ttmv.ranks_of(ref))
        assert np.linalg.norm(ttmv.full(out) - H) <= tol * np.linalg.norm(H)


def test_P38_orthogonalization_invariants():
    cores = _rand_tt((5, 6, 7, 11), (3, 4, 5), 39)
    T = ttmv.full(cores)
    G = ttround.orthogonalize_rl(cores)
    assert np.linalg.norm(ttmv.full(G) - T) <= 1e-13 * np.linalg.norm(T)
    for k in range(1, 4):
        a, n, b = G[k].shape
        R = G[k].reshape((a, n * b), order="F")
        assert np.allclose(R @ R.conj().T, np.eye(a), atol=1e-13)
    assert abs(np.linalg.norm(G[0]) - np.linalg.norm(T)) <= 1e-13 * np.linalg.norm(T)
    # Gram-chain norm / inner product / difference vs the dense tensor
    other = _rand_tt((5, 6, 7, 11), (2, 2, 3), 40)
    T2 = ttmv.full(other)
    assert abs(ttround.tt_norm(cores) - np.linalg.norm(T)) <= 1e-12 * np.linalg.norm(T)
    assert abs(ttround.tt_inner(cores, other) - np.vdot(T2, T)) <= 1e-12 * np.linalg.norm(T) * np.linalg.norm(T2)
    assert abs(ttround.tt_diff_norm(cores, other) - np.linalg.norm(T - T2)) <= 1e-13 * np.linalg.norm(T)
    # close tensors: the difference norm keeps its digits (no sqrt(u) cancellation floor)
    near = [c.copy() for c in cores]
    near[3] = near[3] * (1 + 1e-11)
    assert abs(ttround.tt_diff_norm(cores, near) - 1e-11 * np.linalg.norm(T)) <= 1e-3 * 1e-11 * np.linalg.norm(T)


def test_P39_round_special_cases_and_idempotence():
    dims = (5, 6, 7, 8)
    vs = [np.random.default_rng(k).normal(size=d) + 1j for k, d in enumerate(dims)]
    rank1 = _inflate([v.reshape((1, -1, 1)).astype(complex) for v in vs], 4, 41)
    out = ttround.tt_round(rank1, 1e-12)
    assert ttmv.ranks_of(out) == (1, 1, 1)
    S = np.einsum("i,j,k,l->ijkl", *vs)
    assert np.linalg.norm(ttmv.full(out) - S) <= 1e-13 * np.linalg.norm(S)
    zero = [np.zeros((1 if k == 0 else 3, d, 1 if k == 3 else 3), complex) for k, d in enumerate(dims)]
    z = ttround.tt_round(zero, 1e-6)
    assert ttmv.ranks_of(z) == (1, 1, 1) and np.all(ttmv.full(z) == 0)
    cores = _rand_tt(dims, (3, 4, 3), 42)
    once = ttround.tt_round(cores, 1e-8)
    twice = ttround.tt_round(once, 1e-8)
    assert ttmv.ranks_of(once) == ttmv.ranks_of(twice)
    T1 = ttmv.full(once)
    assert np.linalg.norm(ttmv.full(twice) - T1) <= 1e-12 * np.linalg.norm(T1)


# ---------------------------------------------------------------- PWL test moments (NEXT-2)

def _one_rwg_mesh(D):
    xyz = np.array([[0, -0.01, 0], [0, 0.01, 0], [0.015, 0, 0.002], [-0.012, 0.001, 0]], dtype=float)
    tri = np.array([[0, 1, 2], [1, 0, 3]], dtype=np.int32)
    return xyz + D * np.array([0.8, 0.5, -0.33]), tri


def _one_rwg_problem(D, moment, ng=2, h=(3e-3, 4e-3, 5e-3), origin=(0.0, 0.0, 0.0)):
    shifted, tri = _one_rwg_mesh(D)
    return entries.make_problem((1, 1, 1), h, origin, [(shifted, tri)], 298e6, ng=ng, moment=moment)


def test_P40_pwl_one_point_rule_neglects_linear_terms(cfg1):
    """P:381 / P:287: with one volume node per voxel the linear PWL blocks vanish
    identically (the node sits at the centre, where (r - c)_l = 0), while the PWC block
    equals the midpoint rule V f(c)."""
    meshes = cfg1.meshes()
    rows = np.arange(0, 3 * cfg1.n_v, 997)
    cols = (rows * 7) % (sum(len(t) for _, t in meshes) // 2)
    for l in (1, 2, 3):
        p = entries.make_problem(cfg1.n, cfg1.h, cfg1.origin, meshes, cfg1.freq, ng=1, moment=l)
        assert np.all(entries.entries(p, rows, cols) == 0)
    p0 = entries.make_problem(cfg1.n, cfg1.h, cfg1.origin, meshes, cfg1.freq, ng=1)
    assert np.all(np.abs(entries.entries(p0, rows, cols)) > 0)
    with pytest.raises(ValueError):
        entries.make_problem(cfg1.n, cfg1.h, cfg1.origin, meshes, cfg1.freq, moment=4)


def test_P41_pwl_moment_is_h_over_12_times_centre_gradient():
    """Taylor expansion of the integrand f about the voxel centre c: the odd parts of
    (r - c)_l / h_l f(r) integrate to zero and int_V ((r - c)_l)^2 / h_l = V h_l / 12, so
    Z_l(c) = (h_l / 12) d/dc_l Z_0(c) + O((h / D)^2) relative, with D the source distance.
    The derivative is a central difference of the PWC entry in the voxel origin (an
    independent route through the PWC arithmetic).  Anisotropic h catches an axis mix-up,
    the sign of the difference a sign error, the h_l / 12 factor a scale error; the error
    must fall ~ D^-2."""
    h = (3e-3, 4e-3, 5e-3)
    errs = []
    for D in (0.05, 0.1, 0.2):
        for l in (1, 2, 3):
            Zl = entries.field_vectors(_one_rwg_problem(D, l, h=h), [0], [0])[0]
            dlt = 1e-3 * h[l - 1]
            e = np.zeros(3)
            e[l - 1] = dlt
            Zp = entries.field_vectors(_one_rwg_problem(D, 0, h=h, origin=tuple(e)), [0], [0])[0]
            Zm = entries.field_vectors(_one_rwg_problem(D, 0, h=h, origin=tuple(-e)), [0], [0])[0]
            pred = h[l - 1] / 12.0 * (Zp - Zm) / (2 * dlt)
            errs.append((D, l, np.max(np.abs(Zl - pred)) / np.max(np.abs(pred))))
    by_d = {}
    for D, l, e in errs:
        by_d[D] = max(by_d.get(D, 0.0), e)
    ds = sorted(by_d)
    assert by_d[ds[-1]] < 0.5 * (max(h) / ds[-1]) ** 2, errs   # O((h / D)^2)
    for a, b in zip(ds, ds[1:]):
        assert 2.5 < by_d[a] / by_d[b] < 6.0, by_d    # ~4 per doubling of D


def test_P42_two_surface_column_order():
    """SURVEY §8c-L10 (surfaces concatenated in input order, shield then bore) pinned by the
    geometry itself, not by the GPU: every interior-rule source node of an RWG on a cylinder of
    radius R with N_az azimuthal cells lies inside the chord polygon band
    R cos(pi / N_az) <= r_xy <= R and |z| <= L / 2, and the shield (R 0.34, L 1.2) and bore
    (R 0.40, L 2.0) bands are disjoint -- so the first 14960 columns of cfg 3 are exactly the
    shield RWGs (N_az (3 N_ax - 1) = 88 x 170) and the last 15040 the bore RWGs (80 x 188).  The
    combined table also equals the single-surface problems' tables, column for column."""
    cfg = synth.get_config(3)
    meshes = cfg.meshes()
    rs, js = geometry.mesh_sources(meshes)
    sh, bo = cfg.surfaces
    ns, nb = sh.n_rwg, bo.n_rwg
    assert (ns, nb) == (14960, 15040) and rs.shape[0] == ns + nb
    rad = np.hypot(rs[..., 0], rs[..., 1])
    for sl, s in ((slice(0, ns), sh), (slice(ns, ns + nb), bo)):
        r = rad[sl]
        assert r.max() <= s.radius * (1 + 1e-12)
        assert r.min() >= s.radius * np.cos(np.pi / s.n_az) * (1 - 1e-12)
        assert np.abs(rs[sl][..., 2]).max() <= s.length / 2 * (1 + 1e-12)
    assert sh.radius < bo.radius * np.cos(np.pi / bo.n_az)       # the bands do not overlap
    for sl, msh in ((slice(0, ns), meshes[0]), (slice(ns, ns + nb), meshes[1])):
        r1, j1 = geometry.mesh_sources([msh])
        assert np.array_equal(rs[sl], r1) and np.array_equal(js[sl], j1)


def test_P35b_compression_factor_counts_arrays():
    """The compression factor's numerator / denominator are the element counts of the dense
    tensor (built by the oracle's dense expansion) and of the core arrays themselves, on a
    small random TT -- not a retyped formula."""
    from gpu_common import rand_cores
    n, m = (3, 4, 5), 6
    ranks = [(2, 3, 2), (1, 2, 3), (3, 1, 1)]
    tts = [rand_cores(n + (m,), r, 11 + c) for c, r in enumerate(ranks)]
    dense = ttmv.full_matrix(tts)
    assert dense.shape == (3 * 3 * 4 * 5, m)
    f = validate.compression_factor(n, m, ranks)
    assert f == Fraction(dense.size, sum(g.size for t in tts for g in t))


# ---------------------------------------------------------------- far-near block (NEXT-3)

def _farnear_tables(ci):
    from oracle import farnear  # noqa: F401
    cfg = synth.get_config(ci)
    rs_n, js_n = geometry.mesh_sources([synth.near_mesh(ci)])
    rs_f, js_f = geometry.mesh_sources(cfg.meshes())
    return cfg, rs_n, js_n, rs_f, js_f


def _mp_cc_entry(near, far, m, n):
    """One Z_cc^fn entry at 40 digits from f = +-(l / 2A) (r - p) on each triangle, area weights
    A / 3 on both sides, and the dyad (I + grad grad / k0^2) g by mpmath derivatives of g (no
    closed-form dyad)."""
    mp.mp.dps = 40
    k0 = 2 * mp.pi * mp.mpf(synth.configs.FREQ_7T) / mp.mpf(synth.configs.C0)

    def rwg_nodes(mesh, idx):
        xyz, tri = mesh
        rwg = geometry.rwg_edges(xyz, tri)
        tp, tm = int(rwg["tp"][idx]), int(rwg["tm"][idx])
        a, b = int(rwg["a"][idx]), int(rwg["b"][idx])
        P = lambda v: [mp.mpf(float(x)) for x in v]
        l = mp.sqrt(sum((P(xyz[a])[i] - P(xyz[b])[i]) ** 2 for i in range(3)))
        out = []
        for sgn, T in ((1, tp), (-1, tm)):
            V = [P(xyz[v]) for v in tri[T]]
            p = [P(xyz[v]) for v in tri[T] if v not in (a, b)][0]
            e1 = [V[1][i] - V[0][i] for i in range(3)]
            e2 = [V[2][i] - V[0][i] for i in range(3)]
            cr = [e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]]
            A = mp.sqrt(sum(x * x for x in cr)) / 2
            for q in range(3):
                bary = [mp.mpf(1) / 6] * 3
                bary[q] = mp.mpf(2) / 3
                rq = [sum(bary[j] * V[j][i] for j in range(3)) for i in range(3)]
                f = [sgn * l / (2 * A) * (rq[i] - p[i]) for i in range(3)]
                out.append((rq, [A / 3 * fi for fi in f]))
        return out

    def g(x, y, z):
        rr = mp.sqrt(x * x + y * y + z * z)
        return mp.exp(-1j * k0 * rr) / (4 * mp.pi * rr)

    total = mp.mpc(0)
    for rp, jp in rwg_nodes(near, m):
        for rs, js in rwg_nodes(far, n):
            R = [rp[i] - rs[i] for i in range(3)]
            g0 = g(*R)
            for a in range(3):
                for b in range(3):
                    order = [0, 0, 0]
                    order[a] += 1
                    order[b] += 1
                    Gab = (g0 if a == b else 0) + mp.diff(g, R, tuple(order)) / k0 ** 2
                    total += jp[a] * Gab * js[b]
    return complex(total)


def test_P44_farnear_entry_extended_precision():
    from oracle import farnear
    cfg, rs_n, js_n, rs_f, js_f = _farnear_tables(1)
    k0 = 2 * np.pi * cfg.freq / synth.configs.C0
    for m, n in ((3, 17), (200, 1000)):
        ref = _mp_cc_entry(synth.near_mesh(1), cfg.meshes()[0], m, n)
        got = farnear.entries_cc(rs_n, js_n, rs_f, js_f, k0, [m], [n])[0]
        assert abs(got - ref) <= 1e-13 * abs(ref), (m, n, got, ref)


def test_P43_farnear_reciprocity_and_disjointness():
    """Z^nf = (Z^fn)^T (the dyad is symmetric and even: the transposed block of Eq. 11 / 15),
    and the near and far conductors are disjoint (non-singular rule)."""
    from oracle import farnear
    cfg, rs_n, js_n, rs_f, js_f = _farnear_tables(1)
    k0 = 2 * np.pi * cfg.freq / synth.configs.C0
    rng = np.random.default_rng(43)
    rows = rng.integers(0, rs_n.shape[0], 50)
    cols = rng.integers(0, rs_f.shape[0], 50)
    a = farnear.entries_cc(rs_n, js_n, rs_f, js_f, k0, rows, cols)
    b = farnear.entries_cc(rs_f, js_f, rs_n, js_n, k0, cols, rows)
    assert np.max(np.abs(a - b)) <= 1e-14 * np.max(np.abs(a))
    d = np.min(np.linalg.norm(rs_n.reshape(-1, 1, 3) - rs_f.reshape(1, -1, 3)[:, ::7], axis=-1))
    assert d > 0.15


def test_P45_aca_exact_on_low_rank_and_interpolates_pivots():
    """A seeded random rank-5 complex 60 x 80 matrix is recovered to 1e-12 with rank <= 6; the
    ACA residual vanishes on the pivot rows and columns (cross interpolation)."""
    from oracle import farnear
    rng = np.random.default_rng(45)
    A = (rng.standard_normal((60, 5)) + 1j * rng.standard_normal((60, 5))) @ \
        (rng.standard_normal((5, 80)) + 1j * rng.standard_normal((5, 80)))
    U, W = farnear.aca(lambda i: A[i], lambda j: A[:, j], 60, 80, 1e-14)
    assert U.shape[1] <= 6
    assert np.linalg.norm(A - U @ W.T) <= 1e-12 * np.linalg.norm(A)
    B = rng.standard_normal((40, 30)) + 1j * rng.standard_normal((40, 30))   # full rank
    U, W = farnear.aca(lambda i: B[i], lambda j: B[:, j], 40, 30, 1e-3, max_rank=7)
    Rz = B - U @ W.T
    piv_cols = [int(np.argmax(np.abs(W[:, k]))) for k in range(W.shape[1])]
    assert np.max(np.abs(Rz[:, piv_cols])) <= 1e-12 * np.max(np.abs(B))
    # replaying the run's own (row, column) pivots reproduces it with unit pivot ratios, and the
    # residual vanishes on the pivot rows too
    rows, cols = [], []
    U0, W0 = farnear.aca(lambda i: (rows.append(i), B[i])[1], lambda j: (cols.append(j), B[:, j])[1], 40, 30, 1e-3,
                         max_rank=7)
    assert np.max(np.abs(Rz[rows])) <= 1e-12 * np.max(np.abs(B))
    tr = []
    U1, W1 = farnear.aca(lambda i: B[i], lambda j: B[:, j], 40, 30, 1e-3, max_rank=7, pivots=list(zip(rows, cols)),
                         trace=tr)
    assert np.array_equal(U0, U1) and np.array_equal(W0, W1)
    assert len(tr) == 7 and all(abs(a - 1) <= 1e-12 and abs(b - 1) <= 1e-12 for a, b in tr), tr


def test_P46_aca_far_near_block_vs_dense():
    """The ACA of the cfg 1 far-near block (368 near x 1128 far RWG) meets its tolerance
    against the dense block, and is near the SVD-optimal rank."""
    from oracle import farnear
    cfg, rs_n, js_n, rs_f, js_f = _farnear_tables(1)
    k0 = 2 * np.pi * cfg.freq / synth.configs.C0
    Z = farnear.dense_cc(rs_n, js_n, rs_f, js_f, k0)
    tol = 1e-6
    U, W = farnear.aca(lambda i: Z[i], lambda j: Z[:, j], Z.shape[0], Z.shape[1], tol)
    err = np.linalg.norm(Z - U @ W.T) / np.linalg.norm(Z)
    assert err <= 10 * tol, err
    s = np.linalg.svd(Z, compute_uv=False)
    tail = np.sqrt(np.cumsum((s ** 2)[::-1])[::-1])
    r_opt = int(np.argmax(tail <= tol * np.linalg.norm(Z)))
    assert r_opt <= U.shape[1] <= 2 * r_opt + 10, (r_opt, U.shape[1])
    x = synth.complex_gaussian(Z.shape[1], 46)
    assert np.linalg.norm(farnear.apply_lowrank(U, W, x, "N") - Z @ x) <= 10 * tol * np.linalg.norm(Z) * np.linalg.norm(x)


# ---------------------------------------------------------------- far-far block (NEXT-3)

def _duffy(V, r, fn, order=48):
    """int_T fn(r') dS' by splitting T into the signed sub-triangles (rho, V_i, V_i+1) about the
    in-plane projection rho of r and a Duffy map r' = rho + u (d_i + v e_i), dS' = 2 A_i u du dv
    (the 1/R singularity at rho is cancelled by the Jacobian), Gauss-Legendre order x order."""
    V = np.asarray(V, dtype=np.float64)
    n = np.cross(V[1] - V[0], V[2] - V[0])
    n /= np.linalg.norm(n)
    h = (r - V[0]) @ n
    rho = r - h * n
    x, w = np.polynomial.legendre.leggauss(order)
    x = 0.5 * (x + 1)
    w = 0.5 * w
    U, Vv = np.meshgrid(x, x, indexing="ij")
    WW = np.outer(w, w)
    tot = 0
    for i in range(3):
        a, b = V[i], V[(i + 1) % 3]
        d, e = a - rho, b - a
        A2 = np.cross(d, e) @ n                     # 2 x signed area
        P = rho + U[..., None] * (d + Vv[..., None] * e)
        tot = tot + np.tensordot(WW * U * A2, fn(P), axes=([0, 1], [0, 1]))
    return tot


def test_P47_triangle_potentials_vs_duffy_quadrature():
    """Closed-form I0 = int 1/R and I1 = int (r' - r)/R over a flat triangle against Duffy-mapped
    Gauss quadrature: points in the plane (inside, at a quadrature node, outside, on a vertex, on
    an edge) and off the plane."""
    from oracle import farfar
    rng = np.random.default_rng(47)
    for trial in range(4):
        V = rng.standard_normal((3, 3)) * 0.03
        L = farfar.longest_edge(V)
        n = np.cross(V[1] - V[0], V[2] - V[0])
        n /= np.linalg.norm(n)
        c = V.mean(axis=0)
        pts = [c, V.T @ np.array([2 / 3, 1 / 6, 1 / 6]), c + 1.5 * (V[0] - c), V[1], 0.5 * (V[1] + V[2]),
               c + 0.3 * L * n, V[2] + 0.05 * L * n, c + 2 * (V[1] - c) - 0.7 * L * n]
        for r in pts:
            I0, I1 = farfar.tri_potentials(V, r[None])
            q0 = _duffy(V, r, lambda P: 1.0 / np.linalg.norm(P - r, axis=-1), order=160)
            q1 = _duffy(V, r, lambda P: (P - r) / np.linalg.norm(P - r, axis=-1)[..., None], order=160)
            assert abs(I0[0] - q0) <= 1e-12 * abs(q0), (trial, r, I0, q0)
            assert np.max(np.abs(I1[0] - q1)) <= 1e-12 * np.max(np.abs(q1)), (trial, I1, q1)


def _ff_tables(ci):
    from oracle import farfar
    cfg = synth.get_config(ci)
    return cfg, farfar.rwg_triangle_tables(cfg.meshes()), 2 * np.pi * cfg.freq / synth.configs.C0


def test_P48_near_pair_integral_within_rule_error():
    """The near-pair K (analytic 1/R part + 3-point g_s remainder) against the same integral
    with the inner integral done by Duffy-mapped Gauss quadrature of the full integrand: they
    differ only by the 3-point rule's error on the bounded remainder g_s, which is
    O((k0 L)^2) smaller than the 1/R part -- bound 0.01 (k0 L)^2 of |K| (measured 1.3e-4 self,
    1.7e-5 adjacent at k0 L = 0.24), checked on the self pair and an edge-adjacent pair of cfg 2's
    shield; the plain 3 x 3 rule misses the adjacent pair by > 1 % (the subtraction matters)."""
    from oracle import farfar
    cfg, T, k0 = _ff_tables(2)
    for (m, sm), (n, sn) in (((0, "p"), (0, "p")), ((5, "p"), (5, "m")), ((7, "m"), (40, "p"))):
        Va, pa = T["V" + sm][m], T["p" + sm][m]
        Vb, pb = T["V" + sn][n], T["p" + sn][n]
        if not farfar.is_near(Va, Vb):
            continue
        K = farfar.k_near_oneway(Va, pa, Vb, pb, k0)
        ra = np.einsum("qj,jc->qc", geometry.TRI_BARY, Va)
        ref = 0
        for q in range(3):
            f = lambda P, q=q: ((P - pb) @ (ra[q] - pa) - 4 / k0 ** 2) * np.exp(
                -1j * k0 * np.linalg.norm(P - ra[q], axis=-1)) / (4 * np.pi * np.linalg.norm(P - ra[q], axis=-1))
            ref += farfar.tri_area(Va) / 3 * _duffy(Vb, ra[q], f, order=48)
        kL = k0 * max(farfar.longest_edge(Va), farfar.longest_edge(Vb))
        assert abs(K - ref) <= 0.01 * kL ** 2 * abs(ref), (m, n, K, ref, kL)
        if m != n or sm != sn:
            assert abs(farfar.k_regular(Va, pa, Vb, pb, k0) - ref) > 0.01 * abs(ref)


def test_P49_farfar_regular_entry_extended_precision():
    """A regular (well separated) Z^ff entry against a 40-digit evaluation of the typed-out
    mixed-potential formula with f = s (l/2A)(r - p), div f = s l / A and the 3 x 3 rule."""
    from oracle import farfar
    cfg, T, k0 = _ff_tables(1)
    mp.mp.dps = 40
    K0 = 2 * mp.pi * mp.mpf(synth.configs.FREQ_7T) / mp.mpf(synth.configs.C0)
    m, n = 600, 3
    Va0, Vb0 = T["Vp"][m], T["Vp"][n]
    assert not farfar.is_near(Va0, Vb0)
    tot = mp.mpc(0)
    P = lambda v: [mp.mpf(float(x)) for x in v]
    for sa, Va, pa in ((1, T["Vp"][m], T["pp"][m]), (-1, T["Vm"][m], T["pm"][m])):
        for sb, Vb, pb in ((1, T["Vp"][n], T["pp"][n]), (-1, T["Vm"][n], T["pm"][n])):
            A = [P(v) for v in Va]
            B = [P(v) for v in Vb]
            area = lambda X: mp.sqrt(sum(c * c for c in [
                (X[1][1] - X[0][1]) * (X[2][2] - X[0][2]) - (X[1][2] - X[0][2]) * (X[2][1] - X[0][1]),
                (X[1][2] - X[0][2]) * (X[2][0] - X[0][0]) - (X[1][0] - X[0][0]) * (X[2][2] - X[0][2]),
                (X[1][0] - X[0][0]) * (X[2][1] - X[0][1]) - (X[1][1] - X[0][1]) * (X[2][0] - X[0][0])])) / 2
            Aa, Ab = area(A), area(B)
            lm, ln_ = mp.mpf(float(T["l"][m])), mp.mpf(float(T["l"][n]))
            PA, PB = P(pa), P(pb)
            for q in range(3):
                wq = [mp.mpf(1) / 6] * 3
                wq[q] = mp.mpf(2) / 3
                rq = [sum(wq[j] * A[j][c] for j in range(3)) for c in range(3)]
                for s in range(3):
                    ws = [mp.mpf(1) / 6] * 3
                    ws[s] = mp.mpf(2) / 3
                    rs = [sum(ws[j] * B[j][c] for j in range(3)) for c in range(3)]
                    fm = [sa * lm / (2 * Aa) * (rq[c] - PA[c]) for c in range(3)]
                    fn = [sb * ln_ / (2 * Ab) * (rs[c] - PB[c]) for c in range(3)]
                    div = (sa * lm / Aa) * (sb * ln_ / Ab)
                    R = mp.sqrt(sum((rq[c] - rs[c]) ** 2 for c in range(3)))
                    g = mp.exp(-1j * K0 * R) / (4 * mp.pi * R)
                    tot += (Aa / 3) * (Ab / 3) * (sum(fm[c] * fn[c] for c in range(3)) - div / K0 ** 2) * g
    got = farfar.entries_ff(T, k0, [m], [n])[0]
    assert abs(got - complex(tot)) <= 1e-13 * abs(complex(tot)), (got, tot)


def test_P50_farfar_symmetry_and_near_rule():
    """Z^ff is symmetric by construction, the diagonal carries the near (singular) rule, and
    the near rule changes a regular pair's K only by the 3-point rule error."""
    from oracle import farfar
    cfg, T, k0 = _ff_tables(1)
    rng = np.random.default_rng(50)
    r = rng.integers(0, len(T["l"]), 40)
    c = rng.integers(0, len(T["l"]), 40)
    assert np.array_equal(farfar.entries_ff(T, k0, r, c), farfar.entries_ff(T, k0, c, r))
    assert farfar.is_near(T["Vp"][3], T["Vp"][3])
    # a pair just outside the near radius: both rules agree to ~ the 3-point error
    Va, pa = T["Vp"][0], T["pp"][0]
    d = np.linalg.norm(T["Vp"].mean(axis=1) - Va.mean(axis=0), axis=1)
    far = np.flatnonzero(~farfar.is_near(np.broadcast_to(Va, T["Vp"].shape), T["Vp"]))
    j = far[np.argmin(d[far])]
    Kr = farfar.k_regular(Va, pa, T["Vp"][j], T["pp"][j], k0)
    Kn = 0.5 * (farfar.k_near_oneway(Va, pa, T["Vp"][j], T["pp"][j], k0)
                + farfar.k_near_oneway(T["Vp"][j], T["pp"][j], Va, pa, k0))
    assert abs(Kr - Kn) <= 2e-3 * abs(Kn), (Kr, Kn)


def test_P51_paper_far_rule_one_by_one():
    """The paper's far-block quadrature ("1 volume and 1 surface integration point"
    for Z_bc^f; oracle quad_rule = 1).  (a) Exactness: the RWG function is linear on each
    triangle, so the centroid rule and the 3-point interior rule integrate it exactly and
    their moment vectors agree: J(centroid) = sum_q J_q(3-point), and the centroid is the
    mean of the 3 interior nodes.  (b) 40 digits: two entries of cfg 1 from the definitions
    (mpmath dyad, centroid weight A, voxel-centre weight h1 h2 h3).  (c) Consistency: shrinking the
    RWG and the voxel by s at a fixed distance, the 1 x 1 rule approaches the 8 x 3 rule at
    first order in s (the RWG function varies by O(1) over its triangles), ~2x per halving;
    a wrong weight would leave an O(1) difference."""
    cfg = synth.get_config(1)
    xyz, tri = cfg.meshes()[0]
    rwg = geometry.rwg_edges(xyz, tri)
    r3, j3 = geometry.source_table(xyz, tri, rwg)
    r1, j1 = geometry.source_table(xyz, tri, rwg, geometry.TRI_CENTROID)
    assert r1.shape[1] == 2 and r3.shape[1] == 6
    assert np.allclose(j1[:, 0], j3[:, :3].sum(axis=1), rtol=0, atol=1e-14 * np.abs(j1).max())
    assert np.allclose(j1[:, 1], j3[:, 3:].sum(axis=1), rtol=0, atol=1e-14 * np.abs(j1).max())
    assert np.allclose(r1[:, 0], r3[:, :3].mean(axis=1), rtol=0, atol=1e-15)
    prob = entries.problem_from_config(cfg, quad_rule=1)
    assert prob.wts.shape == (1,) and np.all(prob.offs == 0)
    for (n, chi, vox) in ((5, 0, (0, 3, 11)), (700, 2, (6, 6, 6))):
        ref = _mp_entry(cfg, n, chi, vox, one_point=True)
        v = vox[0] + cfg.n[0] * (vox[1] + cfg.n[1] * vox[2])
        got = entries.entries(prob, [chi * cfg.n_v + v], [n])[0]
        assert abs(got - ref) <= 1e-14 * abs(ref), (got, ref)
    errs = {}
    for sc in (1.0, 0.5, 0.25, 0.125):
        xyz1, tri1 = _one_rwg_mesh(0.0)
        xyz1 = xyz1 * sc + 0.1 * np.array([0.8, 0.5, -0.33])
        h = tuple(np.array((3e-3, 4e-3, 5e-3)) * sc)
        Z8 = entries.field_vectors(entries.make_problem((1, 1, 1), h, (0.0, 0.0, 0.0), [(xyz1, tri1)], 298e6),
                                   [0], [0])[0]
        Z1 = entries.field_vectors(entries.make_problem((1, 1, 1), h, (0.0, 0.0, 0.0), [(xyz1, tri1)], 298e6,
                                                        quad_rule=1), [0], [0])[0]
        errs[sc] = np.max(np.abs(Z1 - Z8)) / np.max(np.abs(Z8))
    # both rules converge to the same integral; the RWG function varies by O(1) across its
    # triangles, so the 1 x 1 rule's error is first order in the element size (a wrong
    # weight would not converge at all)
    assert errs[1.0] < 0.01, errs
    for a, b in ((1.0, 0.5), (0.5, 0.25), (0.25, 0.125)):
        assert 1.6 < errs[a] / errs[b] < 2.6, errs
    with pytest.raises(ValueError):
        entries.make_problem(cfg.n, cfg.h, cfg.origin, cfg.meshes(), cfg.freq, quad_rule=2)


# ---------------------------------------------------------------- GMRES consumer (NEXT-4)
def test_P52_gmres_textbook_properties():
    """oracle/gmres.py against what the mathematics fixes (Saad & Schultz GMRES; P:287
    tol 1e-5, restart 50): (a) an n x n system is solved in <= n iterations (Krylov space
    exhausts C^n) to the accuracy of numpy.linalg.solve; (b) the Arnoldi relation
    A V_k = V_{k+1} H_k and V_{k+1}^H V_{k+1} = I; (c) the recurrence residual |g_{j+1}| equals
    the true residual ||b - A x_j|| (checked at a cycle end); (d) identity and scaled identity
    converge in one iteration; (e) residuals never increase within a cycle (least squares over
    nested spaces); (f) a restart (m < n) still converges on a well-conditioned system, and
    the zero right-hand side returns x = 0 after 0 iterations."""
    from oracle import gmres
    rng = np.random.default_rng(52)
    n = 40
    A = np.eye(n) * 4 + (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    hist = []
    x, its, rel = gmres.gmres(lambda v: A @ v, b, tol=1e-13, restart=n, max_iter=n, history=hist)
    xs = np.linalg.solve(A, b)
    assert its <= n and np.linalg.norm(x - xs) <= 1e-11 * np.linalg.norm(xs)
    assert all(h1 <= h0 * (1 + 1e-12) for h0, h1 in zip(hist, hist[1:]))
    V, H = gmres.arnoldi(lambda v: A @ v, b, 12)
    assert np.linalg.norm(A @ V[:, :12] - V @ H) <= 1e-13 * np.linalg.norm(A) * np.sqrt(12)
    assert np.linalg.norm(V.conj().T @ V - np.eye(13)) <= 1e-14 * 13
    assert np.allclose(np.triu(H, -1), H)   # upper Hessenberg
    x7, its7, rel7 = gmres.gmres(lambda v: A @ v, b, tol=1e-30, restart=7, max_iter=7)
    assert its7 == 7 and abs(rel7 - np.linalg.norm(b - A @ x7) / np.linalg.norm(b)) <= 1e-12
    for s in (1.0, 2.5 - 1j):
        x1, its1, _ = gmres.gmres(lambda v: s * v, b, tol=1e-12)
        assert its1 == 1 and np.allclose(x1, b / s, rtol=1e-14, atol=0)
    xr, itsr, relr = gmres.gmres(lambda v: A @ v, b, tol=1e-10, restart=5, max_iter=400)
    assert relr <= 1e-10 and np.linalg.norm(b - A @ xr) <= 2e-10 * np.linalg.norm(b)
    x0, its0, rel0 = gmres.gmres(lambda v: A @ v, np.zeros(n), tol=1e-5)
    assert its0 == 0 and not x0.any()


def test_P53_hybrid_operator_blocks():
    """oracle/hybrid.py: the block structure of Eq. 15 -- unit vectors of each unknown group
    pick out the block columns (Z_cc^ff / Z_cc^fn / Z_cb^f for e_f; (Z_cc^fn)^T / Z_cc^nn /
    Z_cb^n for e_n; (Z_cb^f)^T / (Z_cb^n)^T / d_b for e_b), checked against dense copies of
    the TT blocks (ttmv.full_matrix); and the PWC body diagonal is h1 h2 h3 eps_r (Eq. 2)."""
    from oracle import hybrid
    rng = np.random.default_rng(53)
    n, mf, mn = (3, 2, 2), 5, 4
    dims_f, dims_n = n + (mf,), n + (mn,)
    def tt(dims, seed):
        r = np.random.default_rng(seed)
        ranks = (1, 2, 2, 2, 1)
        return [r.normal(size=(ranks[k], dims[k], ranks[k + 1])) + 1j * r.normal(size=(ranks[k], dims[k], ranks[k + 1]))
                for k in range(4)]
    ttf = [tt(dims_f, 10 + c) for c in range(3)]
    ttn = [tt(dims_n, 20 + c) for c in range(3)]
    c = lambda *s: rng.normal(size=s) + 1j * rng.normal(size=s)   # noqa: E731
    blocks = dict(Zff=c(mf, mf), Zfn=c(mn, mf), Znn=c(mn, mn), tt_far=ttf, tt_near=ttn,
                  d_body=hybrid.body_diagonal(n, (1e-3, 2e-3, 3e-3), c(12)))
    assert np.allclose(blocks["d_body"][:12] / 6e-9, blocks["d_body"][12:24] / 6e-9)
    Ff, Fn = ttmv.full_matrix(ttf), ttmv.full_matrix(ttn)      # [3 n_v x m]
    N = mf + mn + 3 * 12
    A = np.column_stack([hybrid.matvec(blocks, e) for e in np.eye(N)])
    ref = np.block([[blocks["Zff"], blocks["Zfn"].T, Ff.T],
                    [blocks["Zfn"], blocks["Znn"], Fn.T],
                    [Ff, Fn, np.diag(blocks["d_body"])]])
    assert np.allclose(A, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
