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


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_apply_modes_agree(ci):
    """The three single-RHS schedules (per-chi chains, persistent dataflow kernel, batched
    kernels) compute the same result (to rounding) for every op; each is bitwise
    reproducible run to run."""
    from paper_2206_12409_b200 import Coupling
    import torch
    cfg = synth.get_config(ci)
    r = cfg.ranks_probe
    ranks = [r, (max(1, r[0] - 1), r[1] + 3, r[2] - 5), (r[0] + 1, max(1, r[1] - 2), r[2] + 7)]
    tts = rand_tts(cfg, ranks, 60 + ci)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    x = _cuda(synth.complex_gaussian(cfg.m, 11))
    u = _cuda(synth.complex_gaussian(3 * cfg.n_v, 12))
    out = {}
    for mode in ("persistent", "chains", "batched"):
        h.configure(mode=mode)
        for op, v in (("N", x), ("T", u), ("C", u)):
            a = h.apply(v, op)
            b = h.apply(v, op)
            assert torch.equal(a, b), (mode, op)
            out[(mode, op)] = a.cpu().numpy()
    for op, v in (("N", x), ("T", u), ("C", u)):
        for mode in ("persistent", "batched"):
            assert validate.rel_l2(out[(mode, op)], out[("chains", op)]) <= 1e-13, (mode, op)
    if ci == 1:
        for op, v in (("N", x), ("T", u), ("C", u)):
            for mode in ("persistent", "chains", "batched"):
                assert validate.rel_l2(out[(mode, op)], ttmv.apply(tts, v.cpu().numpy(), op)) <= TOL


def test_cfg3_full_grid_parity():
    """Config 3 geometry at full size (200 x 120 x 400 voxels, m = 30000 over two
    surfaces) with random cores: r3 > 512 exercises the 256-row-tile GEMV path, n1 = 200
    the long G1 contractions, and every schedule is checked against the oracle (T2)."""
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(3)
    ranks = [(16, 124, 600), (15, 120, 640), (17, 130, 580)]
    tts = rand_tts(cfg, ranks, 303)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    x = synth.complex_gaussian(cfg.m, 31)
    u = synth.complex_gaussian(3 * cfg.n_v, 32)
    ref = {op: ttmv.apply(tts, v, op) for op, v in (("N", x), ("T", u), ("C", u))}
    for mode in ("chains", "batched", "persistent"):
        h.configure(mode=mode)
        for op, v in (("N", x), ("T", u), ("C", u)):
            assert validate.rel_l2(h.apply(_cuda(v), op).cpu().numpy(), ref[op]) <= TOL, (mode, op)


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_apply_pair(ci):
    """vsie_coupling_apply_pair (one GMRES coupling matvec: Z x and Z^T u / Z^H u sharing
    the G4 pass) equals the two separate applies and the oracle; bitwise reproducible."""
    from paper_2206_12409_b200 import Coupling
    import torch
    cfg = synth.get_config(ci)
    r = cfg.ranks_probe
    ranks = [r, (max(1, r[0] - 1), r[1] + 3, r[2] - 5), (r[0] + 1, max(1, r[1] - 2), r[2] + 7)]
    tts = rand_tts(cfg, ranks, 80 + ci)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    x = _cuda(synth.complex_gaussian(cfg.m, 21))
    u = _cuda(synth.complex_gaussian(3 * cfg.n_v, 22))
    for adj in ("T", "C"):
        y, z = h.apply_pair(x, u, adj)
        y2, z2 = h.apply_pair(x, u, adj)
        assert torch.equal(y, y2) and torch.equal(z, z2)
        assert validate.rel_l2(y.cpu().numpy(), h.apply(x, "N").cpu().numpy()) <= 1e-13
        assert validate.rel_l2(z.cpu().numpy(), h.apply(u, adj).cpu().numpy()) <= 1e-13
        if ci == 1:
            assert validate.rel_l2(y.cpu().numpy(), ttmv.apply(tts, x.cpu().numpy(), "N")) <= TOL
            assert validate.rel_l2(z.cpu().numpy(), ttmv.apply(tts, u.cpu().numpy(), adj)) <= TOL


@pytest.mark.parametrize("world", [2, 3])
def test_apply_pair_loopback(dense1, cfg1, world):
    """The pair on the emulated slab partition (collectives around z3 and y4) equals P = 1."""
    from paper_2206_12409_b200 import Coupling
    tts = [ttsvd.tt_svd(ttmv.tensor_of(dense1, cfg1.n, chi), cfg1.tol) for chi in range(3)]
    h1 = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=1)
    hp = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, tts, nrhs_max=1, world=world, loopback=1)
    x = _cuda(synth.complex_gaussian(cfg1.m, 41))
    u = _cuda(synth.complex_gaussian(3 * cfg1.n_v, 42))
    ya, za = h1.apply_pair(x, u, "T")
    yb, zb = hp.apply_pair(x, u, "T")
    assert validate.rel_l2(yb.cpu().numpy(), ya.cpu().numpy()) <= 1e-13
    assert validate.rel_l2(zb.cpu().numpy(), za.cpu().numpy()) <= 1e-13
    assert validate.rel_l2(ya.cpu().numpy(), ttmv.apply(tts, x.cpu().numpy(), "N")) <= TOL


def test_fused_g21_forward(monkeypatch):
    """The opt-in fused forward tail (Y2 = G2 Y3 and y = G1 Y2 in one kernel, Y2 tiles in
    shared memory) matches the oracle; run in a subprocess because the switch is read once."""
    import subprocess, sys, textwrap, os
    code = textwrap.dedent('''
        import sys; sys.path.insert(0, "tests")
        import synth, numpy as np, torch
        from oracle import ttmv, validate
        from gpu_common import grid_of, rand_tts
        from paper_2206_12409_b200 import Coupling
        for ci in (1, 2):
            cfg = synth.get_config(ci)
            tts = rand_tts(cfg, [cfg.ranks_probe] * 3, 90 + ci)
            h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
            x = synth.complex_gaussian(cfg.m, 5)
            y = h.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy()
            assert validate.rel_l2(y, ttmv.apply(tts, x, "N")) <= 1e-12, ci
        print("fused ok")
    ''')
    env = dict(os.environ, VSIE_FUSE_G21="1")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert p.returncode == 0 and "fused ok" in p.stdout, p.stderr[-2000:]


_SCHEDULES = [
    dict(VSIE_PAIR_G4="0"),
    dict(VSIE_PAIR_G4="2", VSIE_SEG_G3="0"),
    dict(VSIE_PAIR_G4="2", VSIE_W2_PARTS="1", VSIE_ZGEMM_CLUSTER="1", VSIE_FWD_TAIL_BATCHED="1", VSIE_G2T="0"),
    dict(VSIE_PAIR_G4="2", VSIE_REDUCE_TMA="1"),
    dict(VSIE_PAIR_G4="2", VSIE_REDUCE_TMA="1", VSIE_RT_CW="8"),
    dict(VSIE_PAIR_G4="2", VSIE_G2T="0", VSIE_ADJ_FUSED="0"),
    dict(VSIE_PAIR_G4="2", VSIE_G2N="1"),
    dict(VSIE_PAIR_G4="2", VSIE_ADJ_FUSED="1"),
    dict(VSIE_PAIR_G4="3"),
    dict(VSIE_PAIR_G4="4"),
    dict(VSIE_PAIR_G4="4", VSIE_W2_PARTS="1", VSIE_REDUCE_TMA="1"),
    dict(VSIE_PAIR_G4="5"),
    dict(VSIE_PAIR_G4="2", VSIE_SINGLE_TMA="0", VSIE_G2T="0"),
    dict(VSIE_PAIR_G4="0", VSIE_REDUCE_REM="0", VSIE_EXPAND_REM="0"),
    dict(VSIE_PAIR_G4="2", VSIE_EXPAND_REM="2"),
    dict(VSIE_PAIR_G4="2", VSIE_FWD_CHAIN_SEG="0"),
    dict(VSIE_PAIR_G4="2", VSIE_G4_CHAIN="1"),
    dict(VSIE_PAIR_G4="2", VSIE_FWD_CHAIN_SEG="1", VSIE_ADJ_CHAIN_SEG="1", VSIE_G2T_CHAIN="1"),
]


@pytest.mark.parametrize("env", _SCHEDULES, ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()))
def test_pair_schedules(env):
    """Every GMRES-pair schedule (VSIE_PAIR_G4: 0 per-chi k_gemv_nt chains, 2 batched TMA G4
    pass with (VSIE_SEG_G3=1) or without the batched TMA G3 steps, 3 six concurrent chains,
    4 every step one batched launch, 5 streaming passes beside the other direction's chains;
    VSIE_W2_PARTS=1 leaves the G2^T split-K partials to the
    G3^T kernel; VSIE_ZGEMM_CLUSTER=0 split-K through global partials instead of the cluster /
    DSMEM reduction; VSIE_ADJ_FUSED=1 the fused G1^T + G2^T kernel k_adj12; VSIE_REDUCE_TMA=1
    the batched TMA-streamed G1^T instead of the per-chi k_reduce_g1; VSIE_FWD_TAIL_BATCHED=1
    the forward's G2 / G1 steps as batched launches; VSIE_G2T=0 the split-K ZGEMM for G2^T
    instead of k_g2t; VSIE_G2N=1 the batched k_g2n for the forward G2 step instead of
    the per-chi ZGEMMs; VSIE_FWD_CHAIN_SEG / VSIE_ADJ_CHAIN_SEG / VSIE_G4_CHAIN the G3 / G4 passes per
    chi in the chains (small rings); VSIE_SINGLE_TMA=0 the per-chi GEMV chains in the single applies)
    equals the oracle matvecs and the separate applies,
    at cfg 1 (ragged ranks) and cfg 2 (several tiles, 148-CTA row blocks); op T and op C.
    Subprocess: the switches are read once per process."""
    import subprocess, sys, textwrap, os
    code = textwrap.dedent('''
        import sys; sys.path.insert(0, "tests")
        import synth, numpy as np, torch
        from oracle import ttmv, validate
        from gpu_common import grid_of, rand_tts
        from paper_2206_12409_b200 import Coupling
        for ci in (1, 2):
            cfg = synth.get_config(ci)
            r = cfg.ranks_probe
            tts = rand_tts(cfg, [r, (r[0] + 1, r[1] - 3, r[2] + 5), (max(1, r[0] - 1), r[1] + 2, r[2] - 7)], 700 + ci)
            h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
            x = synth.complex_gaussian(cfg.m, 51)
            u = synth.complex_gaussian(3 * cfg.n_v, 52)
            xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
            for adj in ("T", "C"):
                y, z = h.apply_pair(xd, ud, adj)
                y2, z2 = h.apply_pair(xd, ud, adj)
                assert torch.equal(y, y2) and torch.equal(z, z2), "not reproducible"
                y, z = y.cpu().numpy(), z.cpu().numpy()
                assert validate.rel_l2(y, h.apply(xd, "N").cpu().numpy()) <= 1e-13, (ci, adj)
                assert validate.rel_l2(z, h.apply(ud, adj).cpu().numpy()) <= 1e-13, (ci, adj)
                if ci == 1 or adj == "T":
                    assert validate.rel_l2(y, ttmv.apply(tts, x, "N")) <= 1e-12, (ci, adj)
                    assert validate.rel_l2(z, ttmv.apply(tts, u, adj)) <= 1e-12, (ci, adj)
        print("schedule ok")
    ''')
    env = dict(os.environ, **env)
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert p.returncode == 0 and "schedule ok" in p.stdout, p.stderr[-2000:]
