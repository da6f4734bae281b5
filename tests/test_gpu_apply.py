"""GPU TT apply (forward / transpose / conjugate transpose, single and block
RHS, loopback slab partition) vs the CPU oracle with identical cores
(relative L2 <= 1e-12 per chi / per RHS column)."""
import numpy as np
import pytest

import synth
from oracle import ttmv, ttsvd, validate

from gpu_common import grid_of, rand_tts

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check_all_ops(h, tts, cfg, nrhs=1, seed=0):
    nv = cfg.n_v
    if nrhs == 1:
        x = synth.complex_gaussian(cfg.m, synth.SEEDS["x"] + seed)
        u = synth.complex_gaussian(3 * nv, synth.SEEDS["u"] + seed)
    else:
        x = synth.complex_gaussian(cfg.m, synth.SEEDS["X"] + seed, ncols=nrhs)
        u = synth.complex_gaussian(3 * nv, synth.SEEDS["U"] + seed, ncols=nrhs)
    y = h.apply(_cuda(x), "N").cpu().numpy()
    yr = ttmv.apply(tts, x, "N")
    yr2 = yr.reshape(3, nv, -1) if nrhs > 1 else yr.reshape(3, nv)
    y2 = y.reshape(3, nv, -1) if nrhs > 1 else y.reshape(3, nv)
    for chi in range(3):                                  # per chi (and per column)
        if nrhs == 1:
            assert validate.rel_l2(y2[chi], yr2[chi]) <= TOL
        else:
            for j in range(nrhs):
                assert validate.rel_l2(y2[chi][:, j], yr2[chi][:, j]) <= TOL
    for op in ("T", "C"):
        z = h.apply(_cuda(u), op).cpu().numpy()
        zr = ttmv.apply(tts, u, op)
        if nrhs == 1:
            assert validate.rel_l2(z, zr) <= TOL, op
        else:
            for j in range(nrhs):
                assert validate.rel_l2(z[:, j], zr[:, j]) <= TOL, (op, j)
    return x, u


def test_cfg1_ttsvd_cores_vs_oracle_and_dense(dense1, cfg1):
    from paper_2206_12409_b200 import Coupling
    tts = [ttsvd.tt_svd(ttmv.tensor_of(dense1, cfg1.n, chi), cfg1.tol) for chi in range(3)]
    h = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=8)
    x, u = _check_all_ops(h, tts, cfg1)
    # P28: against the dense expansion of the same TT
    Zt = ttmv.full_matrix(tts)
    assert validate.rel_l2(h.apply(_cuda(x), "N").cpu().numpy(), Zt @ x) <= TOL
    assert validate.rel_l2(h.apply(_cuda(u), "T").cpu().numpy(), Zt.T @ u) <= TOL
    # exported cores are the imported ones, bit for bit
    ex = h.export_cores()
    for chi in range(3):
        for k in range(4):
            assert np.array_equal(ex[chi][k], tts[chi][k])


def test_cfg1_block_rhs_equals_single(dense1, cfg1):
    from paper_2206_12409_b200 import Coupling
    import torch
    tts = [ttsvd.tt_svd(ttmv.tensor_of(dense1, cfg1.n, chi), cfg1.tol) for chi in range(3)]
    h = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=8)
    X, U = _check_all_ops(h, tts, cfg1, nrhs=8, seed=3)
    Y = h.apply(_cuda(X), "N").cpu().numpy()
    Z = h.apply(_cuda(U), "T").cpu().numpy()
    for j in range(8):                                     # P31
        yj = h.apply(_cuda(X[:, j]), "N").cpu().numpy()
        zj = h.apply(_cuda(U[:, j]), "T").cpu().numpy()
        assert validate.rel_l2(Y[:, j], yj) <= 1e-13
        assert validate.rel_l2(Z[:, j], zj) <= 1e-13
    # determinism: bitwise identical on repeat
    assert torch.equal(h.apply(_cuda(X[:, 0]), "N"), h.apply(_cuda(X[:, 0]), "N"))


@pytest.mark.parametrize("ci", [2, 4])
def test_full_size_probe_ranks(ci):
    """Random cores at the config's probe ranks and full sizes (ragged tiles everywhere)."""
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(ci)
    r = cfg.ranks_probe
    ranks = [r, (r[0] - 1, r[1] - 3, r[2] + 5), (r[0] + 1, r[1] + 2, r[2] - 7)]
    tts = rand_tts(cfg, ranks, 40 + ci)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=2)
    _check_all_ops(h, tts, cfg)


def test_expansion_balanced_partition_ragged():
    """The G1 expansion's balanced warp partition (contiguous (task, i1 tile) unit ranges, used
    when whole-task rounds would leave > 10% of the kernel idle: here 5344 column tasks on at most
    3552 warps = 1.5 rounds) on a grid with a ragged column tail (42750 = 8 * 5343 + 6) and a
    ragged i1 tile (n1 = 13), for r1 % 4 = 2, 1 and 0, vs the oracle (T2, 1e-12)."""
    import dataclasses
    from paper_2206_12409_b200 import Coupling
    c1 = synth.get_config(1)
    n = (13, 150, 285)
    ext = [c1.n[a] * c1.h[a] for a in range(3)]
    cfg = dataclasses.replace(c1, n=n, h=tuple(ext[a] / n[a] for a in range(3)))
    ranks = [(10, 12, 9), (9, 11, 10), (8, 13, 8)]
    tts = rand_tts(cfg, ranks, 77)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=2)
    _check_all_ops(h, tts, cfg)
    _check_all_ops(h, tts, cfg, nrhs=2, seed=3)


@pytest.mark.parametrize("world", [2, 3, 5])
def test_loopback_slabs_equal_single(dense1, cfg1, world):
    """P33 (emulated on one GPU): the i3-slab / G4-column partition with P ranks
    equals the P = 1 result (the combine order differs only by rounding)."""
    from paper_2206_12409_b200 import Coupling
    tts = [ttsvd.tt_svd(ttmv.tensor_of(dense1, cfg1.n, chi), cfg1.tol) for chi in range(3)]
    h1 = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=4)
    hp = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=4, world=world, loopback=1)
    inf = hp.info()
    assert inf["world"] == world and inf["slab"] == (0, cfg1.n[2]) and inf["cols"] == (0, cfg1.m)
    x = synth.complex_gaussian(cfg1.m, 99)
    u = synth.complex_gaussian(3 * cfg1.n_v, 98)
    for op, v in (("N", x), ("T", u), ("C", u)):
        a = h1.apply(_cuda(v), op).cpu().numpy()
        b = hp.apply(_cuda(v), op).cpu().numpy()
        assert validate.rel_l2(b, a) <= 1e-13
        assert validate.rel_l2(b, ttmv.apply(tts, v, op)) <= TOL
    X = synth.complex_gaussian(cfg1.m, 97, ncols=4)
    assert validate.rel_l2(hp.apply(_cuda(X), "N").cpu().numpy(), ttmv.apply(tts, X, "N")) <= TOL


def test_apply_host_matches_device(dense1, cfg1):
    from paper_2206_12409_b200 import Coupling
    tts = [ttsvd.tt_svd(ttmv.tensor_of(dense1, cfg1.n, chi), cfg1.tol) for chi in range(3)]
    h = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=4)
    x = synth.complex_gaussian(cfg1.m, 5)
    u = synth.complex_gaussian(3 * cfg1.n_v, 6)
    assert np.array_equal(h.apply_host(x, "N"), h.apply(_cuda(x), "N").cpu().numpy())
    assert np.array_equal(h.apply_host(u, "C"), h.apply(_cuda(u), "C").cpu().numpy())
    assert np.all(h.apply_host(np.zeros(cfg1.m, complex), "N") == 0)   # P30


@pytest.mark.parametrize("ci", [1, 2])
def test_apply_pair_host(ci):
    """The host-buffer pair (forward copy-out overlapped with the transpose's copy-in on two
    streams) equals the device pair and the separate applies, repeatedly (workspaces of the
    two concurrent directions are disjoint), for op T and op C."""
    from paper_2206_12409_b200 import Coupling
    import torch
    cfg = synth.get_config(ci)
    r = cfg.ranks_probe
    tts = rand_tts(cfg, [r, (r[0] + 1, r[1] - 2, r[2] + 3), (max(1, r[0] - 1), r[1] + 1, r[2] - 4)], 300 + ci)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    x = synth.complex_gaussian(cfg.m, 31)
    u = synth.complex_gaussian(3 * cfg.n_v, 32)
    for adj in ("T", "C"):
        yd, zd = h.apply_pair(_cuda(x), _cuda(u), adj)
        yd, zd = yd.cpu().numpy(), zd.cpu().numpy()
        for _ in range(3):
            yh, zh = h.apply_pair_host(x, u, adj)
            assert validate.rel_l2(yh, yd) <= 1e-13 and validate.rel_l2(zh, zd) <= 1e-13
        assert validate.rel_l2(zh, h.apply(_cuda(u), adj).cpu().numpy()) <= 1e-13
        if ci == 1:
            assert validate.rel_l2(yh, ttmv.apply(tts, x, "N")) <= TOL
            assert validate.rel_l2(zh, ttmv.apply(tts, u, adj)) <= TOL


def test_tt_eval_matches_oracle(cfg1):
    from paper_2206_12409_b200 import Coupling
    import torch
    tts = rand_tts(cfg1, [(3, 5, 7), (2, 4, 6), (4, 4, 4)], 77)
    h = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=1)
    idx = synth.uniform_indices(tuple(cfg1.n) + (cfg1.m,), 500, 5)
    for chi in range(3):
        v = idx[:, 0] + cfg1.n[0] * (idx[:, 1] + cfg1.n[1] * idx[:, 2])
        got = h.tt_eval(torch.from_numpy(chi * cfg1.n_v + v), torch.from_numpy(idx[:, 3])).cpu().numpy()
        ref = ttmv.eval_at(tts[chi], idx)
        assert validate.rel_l2(got, ref) <= 1e-13


def _pair_check(h, tts, cfg, x, u, oracle=True):
    """apply_pair under every schedule: bitwise reproducible, equal to the separate applies
    (1e-13) and, with `oracle`, to the oracle TT matvecs (T2, 1e-12), op T and op C."""
    import torch
    xd, ud = _cuda(x), _cuda(u)
    ref = {op: ttmv.apply(tts, v, op) for op, v in (("N", x), ("T", u), ("C", u))} if oracle else None
    sep = {op: h.apply(v, op).cpu().numpy() for op, v in (("N", xd), ("T", ud), ("C", ud))}
    for sched in ("g4_shared", "g3_shared"):
        h.configure(pair_schedule=sched)
        assert h.info()["pair_schedule"] == sched
        for adj in ("T", "C"):
            y, z = h.apply_pair(xd, ud, adj)
            y2, z2 = h.apply_pair(xd, ud, adj)
            assert torch.equal(y, y2) and torch.equal(z, z2), (sched, adj)
            y, z = y.cpu().numpy(), z.cpu().numpy()
            assert validate.rel_l2(y, sep["N"]) <= 1e-13, (sched, adj)
            assert validate.rel_l2(z, sep[adj]) <= 1e-13, (sched, adj)
            if oracle:
                assert validate.rel_l2(y, ref["N"]) <= TOL, (sched, adj)
                assert validate.rel_l2(z, ref[adj]) <= TOL, (sched, adj)
    h.configure(pair_schedule="auto")
    return ref


def test_cfg3_build_ranks_pair_and_applies():
    """Config 3 geometry at full size (200 x 120 x 400 voxels, m = 30000 over shield + bore)
    with random cores at the ranks of the cfg 3 TT-cross build (r3 ~ 1500 > 320: the row-band
    G4 pass and the large-C G3 passes; r1 = 17: the DFMA remainder of the G1 steps).  Single
    applies N / T / C and the pair under both schedules vs the oracle (T2, 1e-12)."""
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(3)
    ranks = [(17, 137, 1541), (16, 128, 1482), (18, 131, 1509)]
    tts = rand_tts(cfg, ranks, 303)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    assert h.info()["pair_schedule"] == "g3_shared"   # |G3| > |G4| at these ranks
    x = synth.complex_gaussian(cfg.m, 31)
    u = synth.complex_gaussian(3 * cfg.n_v, 32)
    ref = _pair_check(h, tts, cfg, x, u)
    for op, v in (("N", x), ("T", u), ("C", u)):
        assert validate.rel_l2(h.apply(_cuda(v), op).cpu().numpy(), ref[op]) <= TOL, op


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_apply_pair(ci):
    """vsie_coupling_apply_pair (one GMRES coupling matvec: Z x and Z^T u / Z^H u sharing
    one pass over G4 or over G3) equals the two separate applies and the oracle; bitwise
    reproducible; both schedules."""
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(ci)
    r = cfg.ranks_probe
    ranks = [r, (max(1, r[0] - 1), r[1] + 3, r[2] - 5), (r[0] + 1, max(1, r[1] - 2), r[2] + 7)]
    tts = rand_tts(cfg, ranks, 80 + ci)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    if ci in (2, 4):
        assert h.info()["pair_schedule"] == "g4_shared"   # |G4| > |G3| at the head configs
    _pair_check(h, tts, cfg, synth.complex_gaussian(cfg.m, 21), synth.complex_gaussian(3 * cfg.n_v, 22))


@pytest.mark.parametrize("world", [2, 3])
def test_apply_pair_loopback(dense1, cfg1, world):
    """The pair on the emulated slab partition (collectives around z3 and y4) equals P = 1."""
    from paper_2206_12409_b200 import Coupling
    tts = [ttsvd.tt_svd(ttmv.tensor_of(dense1, cfg1.n, chi), cfg1.tol) for chi in range(3)]
    h1 = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=1)
    hp = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=1, world=world, loopback=1)
    x = _cuda(synth.complex_gaussian(cfg1.m, 41))
    u = _cuda(synth.complex_gaussian(3 * cfg1.n_v, 42))
    for sched in ("g4_shared", "g3_shared"):
        hp.configure(pair_schedule=sched)
        for adj in ("T", "C"):
            ya, za = h1.apply_pair(x, u, adj)
            yb, zb = hp.apply_pair(x, u, adj)
            assert validate.rel_l2(yb.cpu().numpy(), ya.cpu().numpy()) <= 1e-13, (sched, adj)
            assert validate.rel_l2(zb.cpu().numpy(), za.cpu().numpy()) <= 1e-13, (sched, adj)
            assert validate.rel_l2(ya.cpu().numpy(), ttmv.apply(tts, x.cpu().numpy(), "N")) <= TOL
            assert validate.rel_l2(za.cpu().numpy(), ttmv.apply(tts, u.cpu().numpy(), adj)) <= TOL


def test_cfg5_block_rhs_64_full_size():
    """The block workload at its own shape (BASELINE cfg 5: cfg 3 geometry, m = 30000, random
    cores at the cfg 3 build ranks (17, 137, 1541), nrhs = 64): P31 -- every one of the 64
    columns of the block N / T / C results equals the single-RHS apply of that column (1e-13,
    compared on the device) -- and T2 against the oracle's TT matvec for three columns per op
    (1e-12)."""
    import torch
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(5)
    k = 64
    ranks = [(17, 137, 1541), (16, 128, 1482), (18, 131, 1509)]
    tts = rand_tts(cfg, ranks, 505)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=k)
    X = synth.complex_gaussian(cfg.m, synth.SEEDS["X"], ncols=k)               # host, m x 64
    Xt = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()                    # (64, m): column j = Xt[j]
    g = torch.Generator(device="cuda")
    g.manual_seed(synth.SEEDS["U"])
    Ut = torch.view_as_complex(torch.randn((k, 3 * cfg.n_v, 2), generator=g, device="cuda",
                                           dtype=torch.float64) / np.sqrt(2.0))  # (64, 3 n_v)

    def rel(a, b):
        return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))

    Y = h.apply(Xt.t(), "N")                      # (3 n_v, 64) view of a (64, 3 n_v) block
    for j in range(k):                            # P31, forward
        assert rel(Y[:, j], h.apply(Xt[j], "N")) <= 1e-13, j
    for j in (0, 37, 63):                         # T2 vs the oracle
        yj = Y[:, j].cpu().numpy()
        assert validate.rel_l2(yj, ttmv.apply(tts, X[:, j], "N")) <= TOL, j
    del Y
    for op in ("T", "C"):
        Z = h.apply(Ut.t(), op)                   # (m, 64)
        for j in range(k):
            assert rel(Z[:, j], h.apply(Ut[j], op)) <= 1e-13, (op, j)
        for j in (0, 37, 63):
            uj = Ut[j].cpu().numpy()
            assert validate.rel_l2(Z[:, j].cpu().numpy(), ttmv.apply(tts, uj, op)) <= TOL, (op, j)
