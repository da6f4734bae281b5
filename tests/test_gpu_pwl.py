"""PWL (q = 12) coupling on the GPU (DESIGN.md R-PWL) vs
the CPU oracle's moment entries (oracle.entries.make_problem(moment=l), pinned by P40/P41).

Entry parity is scale-relative (T1's max and L2 criteria at 1e-12): a linear moment is a
signed sum over the 8 nodes that cancels to ~h/D of its terms, so the element-wise
criterion of T1 would measure that cancellation, not the kernel.  The TT path is judged
as for PWC: held-out entries within 10 tol, the applies against the oracle's TT matvec on
the exported cores (1e-12) and the q = 12 transpose against the sum of the four."""
import numpy as np
import pytest

import synth
from oracle import entries as oent
from oracle import ttmv, validate

from gpu_common import grid_of, rand_cores

pytestmark = pytest.mark.gpu


def _scale_rel(got, ref):
    d = np.abs(got - ref)
    return float(d.max() / np.abs(ref).max()), float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


def _moment_problem(cfg, l):
    return oent.make_problem(cfg.n, cfg.h, cfg.origin, cfg.meshes(), cfg.freq, moment=l)


@pytest.mark.parametrize("ci", [1, 2])
def test_moment_entries_vs_oracle(ci):
    import torch
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(ci)
    dims = tuple(cfg.n) + (cfg.m,)
    cores = [rand_cores(dims, (1, 1, 1), 5 + c) for c in range(3)]
    idx = synth.uniform_indices((3 * cfg.n_v, cfg.m), 20_000, 8100 + ci)
    idx[:2] = [[0, 0], [3 * cfg.n_v - 1, cfg.m - 1]]
    for l in range(4):
        h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, cores, nrhs_max=1, test_moment=l)
        assert h.info()["test_moment"] == l
        got = h.entries(torch.from_numpy(idx[:, 0]), torch.from_numpy(idx[:, 1])).cpu().numpy()
        ref = oent.entries(_moment_problem(cfg, l), idx[:, 0], idx[:, 1])
        c1, c2 = _scale_rel(got, ref)
        assert c1 <= 1e-12 and c2 <= 1e-12, (l, c1, c2)
        if l == 0:
            ok, worst = validate.entry_parity(got, ref, tol=1e-12)
            assert ok, worst


def test_bad_moment_rejected(cfg1):
    from paper_2206_12409_b200 import Coupling, VsieError
    dims = tuple(cfg1.n) + (cfg1.m,)
    cores = [rand_cores(dims, (1, 1, 1), 5 + c) for c in range(3)]
    with pytest.raises(VsieError):
        Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cores, test_moment=4)


@pytest.fixture(scope="module")
def pwl1(cfg1):
    from paper_2206_12409_b200 import PWLCoupling
    return PWLCoupling.build(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cfg1.tol, nrhs_max=2)


def test_pwl_build_heldout(pwl1, cfg1):
    """Each moment's TT reproduces fresh oracle entries of that moment within 10 tol."""
    import torch
    idx = synth.uniform_indices((3 * cfg1.n_v, cfg1.m), 5000, 8200)
    for l, h in enumerate(pwl1.handles):
        inf = h.info()
        assert h.status == 0 and inf["test_moment"] == l
        assert max(inf["heldout_err"]) <= 10 * cfg1.tol, (l, inf["heldout_err"])
        tt = h.tt_eval(torch.from_numpy(idx[:, 0]), torch.from_numpy(idx[:, 1])).cpu().numpy()
        ref = oent.entries(_moment_problem(cfg1, l), idx[:, 0], idx[:, 1])
        assert validate.rel_l2(tt, ref) <= 10 * cfg1.tol, l


@pytest.mark.parametrize("nrhs", [1, 2])
@pytest.mark.parametrize("op", ["N", "T", "C"])
def test_pwl_apply_vs_oracle(pwl1, cfg1, op, nrhs):
    import torch
    tts = [h.export_cores() for h in pwl1.handles]
    nvox = 3 * cfg1.n_v
    n_in = cfg1.m if op == "N" else 4 * nvox
    X = np.stack([synth.complex_gaussian(n_in, 8300 + j) for j in range(nrhs)], axis=1)
    xin = torch.from_numpy(X[:, 0] if nrhs == 1 else X).cuda()
    got = pwl1.apply(xin, op).cpu().numpy().reshape(-1, nrhs)
    assert got.shape == (pwl1.out_len(op), nrhs)
    for j in range(nrhs):
        if op == "N":
            ref = np.concatenate([ttmv.apply(tts[l], X[:, j], "N") for l in range(4)])
        else:
            ref = sum(ttmv.apply(tts[l], X[l * nvox:(l + 1) * nvox, j], op) for l in range(4))
        assert validate.rel_l2(got[:, j], ref) <= 1e-12, (op, j)
    # the q = 12 blocks are the four handles' own applies
    if op == "N" and nrhs == 1:
        for l, h in enumerate(pwl1.handles):
            yl = h.apply(xin, "N").cpu().numpy()
            assert validate.rel_l2(got[l * nvox:(l + 1) * nvox, 0], yl) <= 1e-14


def test_pwl_handle_order_checked(pwl1, cfg1):
    import torch
    from paper_2206_12409_b200 import PWLCoupling, VsieError
    bad = PWLCoupling([pwl1.handles[1], pwl1.handles[0], pwl1.handles[2], pwl1.handles[3]])
    with pytest.raises(VsieError):
        bad.apply(torch.zeros(cfg1.m, dtype=torch.complex128, device="cuda"), "N")


@pytest.mark.parametrize("adj", ["T", "C"])
def test_pwl_pair_vs_separate_and_oracle(pwl1, cfg1, adj):
    import torch
    tts = [h.export_cores() for h in pwl1.handles]
    nvox = 3 * cfg1.n_v
    x = synth.complex_gaussian(cfg1.m, 8400)
    u = synth.complex_gaussian(4 * nvox, 8401)
    y, z = pwl1.apply_pair(torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda(), adj)
    y, z = y.cpu().numpy(), z.cpu().numpy()
    yref = np.concatenate([ttmv.apply(tts[l], x, "N") for l in range(4)])
    zref = sum(ttmv.apply(tts[l], u[l * nvox:(l + 1) * nvox], adj) for l in range(4))
    assert validate.rel_l2(y, yref) <= 1e-12
    assert validate.rel_l2(z, zref) <= 1e-12
    ys = pwl1.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy()
    zs = pwl1.apply(torch.from_numpy(u).cuda(), adj).cpu().numpy()
    assert validate.rel_l2(y, ys) <= 1e-13 and validate.rel_l2(z, zs) <= 1e-13


@pytest.mark.parametrize("world", [2, 3])
def test_pwl_pair_loopback_slabs(pwl1, cfg1, world):
    """The slab-sharded PWL pair (i3 planes and G4 columns over `world` ranks, emulated on
    one GPU) equals the single-rank one."""
    import torch
    from paper_2206_12409_b200 import PWLCoupling
    cores4 = [h.export_cores() for h in pwl1.handles]
    hp = PWLCoupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cores4, nrhs_max=1, world=world,
                                loopback=1)
    x = torch.from_numpy(synth.complex_gaussian(cfg1.m, 8500)).cuda()
    u = torch.from_numpy(synth.complex_gaussian(4 * 3 * cfg1.n_v, 8501)).cuda()
    y1, z1 = pwl1.apply_pair(x, u, "T")
    yp, zp = hp.apply_pair(x, u, "T")
    assert validate.rel_l2(yp.cpu().numpy(), y1.cpu().numpy()) <= 1e-13
    assert validate.rel_l2(zp.cpu().numpy(), z1.cpu().numpy()) <= 1e-13
    hp.close()
