"""GPU entry kernel vs the CPU oracle (scale-relative 1e-12).

Calls go through the C ABI (vsie_coupling_entries) on seeded inputs."""
import numpy as np
import pytest

import synth
from oracle import entries as oent
from oracle import validate

from gpu_common import grid_of, rand_cores

pytestmark = pytest.mark.gpu


def _handle(cfg):
    from paper_2206_12409_b200 import Coupling
    dims = tuple(cfg.n) + (cfg.m,)
    cores = [rand_cores(dims, (1, 1, 1), 5 + c) for c in range(3)]
    return Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, cores, nrhs_max=1)


def test_entries_cfg1_all_vs_dense(dense1, cfg1):
    import torch
    h = _handle(cfg1)
    rows, cols = np.meshgrid(np.arange(dense1.shape[0]), np.arange(dense1.shape[1]), indexing="ij")
    got = h.entries(torch.from_numpy(rows.ravel()), torch.from_numpy(cols.ravel())).cpu().numpy()
    ok, worst = validate.entry_parity(got, dense1.ravel(), tol=1e-12)
    assert ok, worst


@pytest.mark.parametrize("ci", [2, 3, 4])
def test_entries_random_sample_full_size(ci):
    import torch
    cfg = synth.get_config(ci)
    h = _handle(cfg)
    prob = oent.problem_from_config(cfg)
    idx = synth.uniform_indices((3 * cfg.n_v, cfg.m), 100_000, 7000 + ci)
    # include the extreme corners (first / last row and column)
    idx[:4] = [[0, 0], [3 * cfg.n_v - 1, cfg.m - 1], [0, cfg.m - 1], [3 * cfg.n_v - 1, 0]]
    got = h.entries(torch.from_numpy(idx[:, 0]), torch.from_numpy(idx[:, 1])).cpu().numpy()
    ref = oent.entries(prob, idx[:, 0], idx[:, 1])
    ok, worst = validate.entry_parity(got, ref, tol=1e-12)
    assert ok, worst


def test_entries_edge_cases(cfg1, prob1):
    import torch
    h = _handle(cfg1)
    out = h.entries(torch.zeros(0, dtype=torch.int64), torch.zeros(0, dtype=torch.int64))
    assert out.numel() == 0
    got = h.entries([5], [7]).cpu().numpy()
    ref = oent.entries(prob1, [5], [7])
    assert abs(got[0] - ref[0]) <= 1e-12 * abs(ref[0])
    # scale option multiplies every entry (reading L4)
    from paper_2206_12409_b200 import Coupling
    dims = tuple(cfg1.n) + (cfg1.m,)
    cores = [rand_cores(dims, (1, 1, 1), 5 + c) for c in range(3)]
    hs = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cores, scale=2.0 - 1.0j)
    got2 = hs.entries([5], [7]).cpu().numpy()
    assert abs(got2[0] - (2 - 1j) * ref[0]) <= 1e-12 * abs(ref[0])


def _block_rc(cfg, chi, k, left, right):
    """Global (row, col) of every element of the column-major supercore M_k:
    rows a + n_left i_k, columns i_{k+1} + n_{k+1} b."""
    n1, n2, n3 = cfg.n
    dims = (n1, n2, n3, cfg.m)
    nl = 1 if left is None else len(left)
    nr = 1 if right is None else len(right)
    R = np.arange(nl * dims[k - 1])
    Cc = np.arange(dims[k] * nr)
    rr, cc = np.meshgrid(R, Cc, indexing="ij")          # element (row, col) of M_k
    a, ik = rr % nl, rr // nl
    ik1, b = cc % dims[k], cc // dims[k]
    if k == 1:
        i1, i2, i3, n = ik, ik1, right[b, 0], right[b, 1]
    elif k == 2:
        i1, i2, i3, n = left[a, 0], ik, ik1, right[b, 0]
    else:
        i1, i2, i3, n = left[a, 0], left[a, 1], ik, ik1
    row = chi * cfg.n_v + i1 + n1 * (i2 + n2 * i3)
    return row.ravel(order="F"), n.ravel(order="F")


@pytest.mark.parametrize("ci,chi,k,nl,nr", [(2, 0, 1, 1, 12), (2, 1, 2, 3, 4), (2, 2, 3, 1, 1), (3, 1, 2, 2, 2),
                                             (1, 2, 3, 8, 1)])
def test_supercore_block_vs_oracle(ci, chi, k, nl, nr):
    """Structured-block entry mode (the TT-cross's black box, vsie_coupling_supercore) vs the
    oracle entries of the same (row, col) pairs, T1 at 1e-12, >= 1e5 entries per block."""
    cfg = synth.get_config(ci)
    h = _handle(cfg)
    prob = oent.problem_from_config(cfg)
    rng = np.random.default_rng(900 + 10 * ci + k)
    n1, n2, n3 = cfg.n
    left = right = None
    if k == 1:
        right = np.stack([rng.integers(0, n3, nr), rng.integers(0, cfg.m, nr)], axis=1).astype(np.int32)
    elif k == 2:
        left = np.stack([rng.integers(0, n1, nl), np.zeros(nl, int)], axis=1).astype(np.int32)
        right = np.stack([rng.integers(0, cfg.m, nr), np.zeros(nr, int)], axis=1).astype(np.int32)
    else:
        left = np.stack([rng.integers(0, n1, nl), rng.integers(0, n2, nl)], axis=1).astype(np.int32)
    got = h.supercore(chi, k, left, right).cpu().numpy().ravel(order="F")
    assert got.size >= 100_000
    rows, cols = _block_rc(cfg, chi, k, left, right)
    ok, worst = validate.entry_parity(got, oent.entries(prob, rows, cols), tol=1e-12)
    assert ok, worst


# ---------------------------------------------------------------- the paper's 1 x 1 far rule
def _handle_rule1(cfg):
    from paper_2206_12409_b200 import Coupling
    dims = tuple(cfg.n) + (cfg.m,)
    cores = [rand_cores(dims, (1, 1, 1), 5 + c) for c in range(3)]
    return Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, cores, nrhs_max=1, quad_rule=1)


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_entries_paper_far_rule(ci):
    """quad_rule = 1 (1 volume x 1 surface point for Z_bc^f) vs the oracle's
    make_problem(quad_rule=1) (pinned by P51) at T1 1e-12: cfg 1 every entry, cfgs 2 / 4
    1e5 uniform random entries + the corners."""
    import torch
    cfg = synth.get_config(ci)
    h = _handle_rule1(cfg)
    assert h.info()["quad_rule"] == 1
    prob = oent.problem_from_config(cfg, quad_rule=1)
    if ci == 1:
        rows, cols = np.meshgrid(np.arange(3 * cfg.n_v), np.arange(cfg.m), indexing="ij")
        rows, cols = rows.ravel(), cols.ravel()
    else:
        idx = synth.uniform_indices((3 * cfg.n_v, cfg.m), 100_000, 7100 + ci)
        idx[:4] = [[0, 0], [3 * cfg.n_v - 1, cfg.m - 1], [0, cfg.m - 1], [3 * cfg.n_v - 1, 0]]
        rows, cols = idx[:, 0], idx[:, 1]
    got = h.entries(torch.from_numpy(rows), torch.from_numpy(cols)).cpu().numpy()
    ref = oent.entries(prob, rows, cols)
    ok, worst = validate.entry_parity(got, ref, tol=1e-12)
    assert ok, worst


def test_entries_paper_far_rule_pwl_moments_vanish(cfg1):
    """P40 on the device: with one volume point the linear PWL test moments are zero."""
    import torch
    from paper_2206_12409_b200 import Coupling
    dims = tuple(cfg1.n) + (cfg1.m,)
    cores = [rand_cores(dims, (1, 1, 1), 5 + c) for c in range(3)]
    h = Coupling.from_cores(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cores, quad_rule=1, test_moment=2)
    rows = np.arange(0, 3 * cfg1.n_v, 37)
    cols = (rows * 11) % cfg1.m
    got = h.entries(torch.from_numpy(rows), torch.from_numpy(cols)).cpu().numpy()
    assert np.all(got == 0)
