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
