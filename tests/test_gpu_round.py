"""GPU TT rounding (vsie_coupling_round) vs the CPU oracle
(oracle/ttround.py, pinned by P36-P39).

What is unique and compared: the ranks (the TT-SVD ranks of the represented tensor,
P37) and the represented tensor (Gram-chain distances, never core equality: the
cores are unique only up to unitary gauge).  Tolerances:
  * redundant-rank removal is exact up to rounding: 1e-12 relative;
  * a rounded TT must be within tol ||A|| of the input (the rounding theorem);
  * GPU vs oracle rounded tensors: both are the same orthogonal projection of A,
    computed by different SVDs (one-sided Jacobi vs LAPACK); their difference is
    bounded by the perturbation of the kept singular subspaces, O(u ||A|| / gap);
    1e-3 tol ||A|| leaves a gap of 1e5 u-relative, checked in practice to hold
    with orders of magnitude to spare."""
import numpy as np
import pytest
import torch

import synth
from oracle import ttmv, ttround, validate

from gpu_common import grid_of, inflate, rand_tts

pytestmark = pytest.mark.gpu


def _from_cores(cfg, tts, **kw):
    from paper_2206_12409_b200 import Coupling
    return Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=2, **kw)


def test_round_removes_redundant_ranks(cfg1):
    ranks = [(3, 5, 4), (2, 7, 6), (4, 4, 9)]
    tts = rand_tts(cfg1, ranks, 5100)
    fat = [inflate(t, 3, 5200 + c) for c, t in enumerate(tts)]
    h = _from_cores(cfg1, fat)
    new = h.round(1e-12)
    assert new == ranks
    out = h.export_cores()
    for chi in range(3):
        nrm = ttround.tt_norm(tts[chi])
        assert ttround.tt_diff_norm(out[chi], tts[chi]) <= 1e-12 * nrm
    x = synth.complex_gaussian(cfg1.m, synth.SEEDS["x"])
    y = h.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy()
    assert validate.rel_l2(y, ttmv.apply(tts, x, "N")) <= 1e-12


def test_round_loopback_shards(cfg1):
    ranks = [(3, 5, 4)] * 3
    tts = rand_tts(cfg1, ranks, 5300)
    fat = [inflate(t, 2, 5400 + c) for c, t in enumerate(tts)]
    h = _from_cores(cfg1, fat, world=2, loopback=1)
    assert h.round(0.0) == ranks
    u = synth.complex_gaussian(3 * cfg1.n_v, synth.SEEDS["u"])
    z = h.apply(torch.from_numpy(u).cuda(), "T").cpu().numpy()
    assert validate.rel_l2(z, ttmv.apply(tts, u, "T")) <= 1e-12


def test_round_zero_tensor(cfg1):
    dims = tuple(cfg1.n) + (cfg1.m,)
    rr = (1, 3, 4, 2, 1)
    tts = [[np.zeros((rr[k], dims[k], rr[k + 1]), complex) for k in range(4)] for _ in range(3)]
    h = _from_cores(cfg1, tts)
    assert h.round(1e-6) == [(1, 1, 1)] * 3
    x = synth.complex_gaussian(cfg1.m, 1)
    y = h.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy()
    assert np.all(y == 0)


@pytest.fixture(scope="module")
def built1(cfg1):
    from paper_2206_12409_b200 import Coupling
    return Coupling.build(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cfg1.tol, nrhs_max=2)


@pytest.mark.parametrize("tol_mult", [1.0, 10.0])
def test_round_cross_output_vs_oracle(cfg1, dense1, tol_mult):
    """The cross TT of config 1 (ranks overestimated) rounded on the GPU and by
    the oracle from the same exported cores: same ranks, tensors within the rounding
    bound of the input and within 1e-3 tol of each other; vs the dense Z the rounded
    TT keeps the build's 10 tol acceptance (+ tol of the rounding)."""
    from paper_2206_12409_b200 import Coupling
    tol = cfg1.tol * tol_mult
    h = Coupling.build(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cfg1.tol, nrhs_max=2)
    src = h.export_cores()
    r_cross = h.info()["ranks"]
    r_gpu = h.round(tol)
    out = h.export_cores()
    for chi in range(3):
        ref = ttround.tt_round(src[chi], tol)
        assert tuple(r_gpu[chi]) == ttmv.ranks_of(ref), (chi, r_gpu[chi], ttmv.ranks_of(ref))
        assert all(a <= b for a, b in zip(r_gpu[chi], r_cross[chi]))
        nrm = ttround.tt_norm(src[chi])
        assert ttround.tt_diff_norm(out[chi], src[chi]) <= tol * nrm
        assert ttround.tt_diff_norm(out[chi], ref) <= 1e-3 * tol * nrm
        A = ttmv.tensor_of(dense1, cfg1.n, chi)
        err = np.linalg.norm(ttmv.full(out[chi]) - A) / np.linalg.norm(A)
        assert err <= 10 * cfg1.tol + tol, (chi, err)


def test_round_cfg2_heldout():
    """Config 2 (BASELINE workload): rounding at tol keeps the held-out acceptance
    (10 tol vs oracle entries) and never raises a rank."""
    from oracle import entries as oent
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(2)
    h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1)
    r0 = h.info()["ranks"]
    r1 = h.round(cfg.tol)
    tts = h.export_cores()
    prob = oent.problem_from_config(cfg)
    s = synth.uniform_indices(tuple(cfg.n) + (cfg.m,), 1000, synth.SEEDS["heldout"])
    v = s[:, 0] + cfg.n[0] * (s[:, 1] + cfg.n[1] * s[:, 2])
    for chi in range(3):
        assert all(a <= b for a, b in zip(r1[chi], r0[chi]))
        ref = oent.entries(prob, chi * cfg.n_v + v, s[:, 3])
        assert validate.rel_l2(ttmv.eval_at(tts[chi], s), ref) <= 10 * cfg.tol
    print("cfg2 ranks cross", r0, "rounded", r1)
