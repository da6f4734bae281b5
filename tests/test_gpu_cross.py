"""GPU TT-cross build (vsie_coupling_build) vs the CPU oracle.

Parity is judged by what is unique (never by pivot or core
equality): reconstruction against the dense oracle Z on config 1 (T3, 10 tol),
held-out entries against oracle entries on the larger configs (T4, 10 tol),
the interpolation property of the cross, and the rank-cap warning path."""
import numpy as np
import pytest

import synth
from oracle import entries as oent
from oracle import ttmv, ttsvd, validate

from gpu_common import grid_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built1(cfg1):
    from paper_2206_12409_b200 import Coupling
    return Coupling.build(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cfg1.tol, nrhs_max=2)


def test_cfg1_reconstruction_vs_dense(built1, dense1, cfg1):
    assert built1.status == 0
    tts = built1.export_cores()
    inf = built1.info()
    for chi in range(3):
        A = ttmv.tensor_of(dense1, cfg1.n, chi)
        err = np.linalg.norm(ttmv.full(tts[chi]) - A) / np.linalg.norm(A)
        assert err <= 10 * cfg1.tol, (chi, err)
        # informational: cross ranks vs TT-SVD ranks (P:389 expects overestimation)
        r_svd = ttmv.ranks_of(ttsvd.tt_svd(A, cfg1.tol))
        r_x = inf["ranks"][chi]
        assert all(a >= b - 2 for a, b in zip(r_x, r_svd)), (r_x, r_svd)
        assert inf["heldout_err"][chi] <= 10 * cfg1.tol
    assert inf["entries_evaluated"] > 0 and inf["compression"] > 1
    dense_elems = 3 * cfg1.n_v * cfg1.m
    tt_elems = ttmv.core_elements(tts)
    assert inf["compression"].numerator * tt_elems == inf["compression"].denominator * dense_elems


def test_cfg1_cores_are_interpolative(built1, cfg1):
    """L->R cores are L L[P]^{-1}; after the final R->L half-sweep G1 holds exact
    fibres A(:, J_{>1}) — the TT reproduces these exact entries."""
    tts = built1.export_cores()
    prob = oent.problem_from_config(cfg1)
    for chi in range(3):
        G1 = tts[chi][0][0]                         # n1 x r1 (exact columns of M_1)
        # the TT evaluated along i1 for a fixed (i2, i3, n) is G1 times a vector:
        # its column space must contain the exact fibres up to 10 tol
        idx = synth.uniform_indices(tuple(cfg1.n) + (cfg1.m,), 20, 300 + chi)
        for t in idx:
            fib = np.array([[i1, t[1], t[2], t[3]] for i1 in range(cfg1.n[0])])
            v = fib[:, 0] + cfg1.n[0] * (fib[:, 1] + cfg1.n[1] * fib[:, 2])
            ex = oent.entries(prob, chi * cfg1.n_v + v, fib[:, 3])
            coef, *_ = np.linalg.lstsq(G1, ex, rcond=None)
            assert np.linalg.norm(G1 @ coef - ex) <= 10 * cfg1.tol * max(np.linalg.norm(ex), 1e-300)


def test_cfg1_apply_with_built_cores(built1, cfg1):
    import torch
    tts = built1.export_cores()
    x = synth.complex_gaussian(cfg1.m, synth.SEEDS["x"])
    y = built1.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy()
    assert validate.rel_l2(y, ttmv.apply(tts, x, "N")) <= 1e-12


def test_rank_cap_returns_warning(cfg1):
    from paper_2206_12409_b200 import Coupling
    h = Coupling.build(grid_of(cfg1), cfg1.meshes(), cfg1.freq, cfg1.tol, max_rank=4, max_sweeps=2, nrhs_max=1)
    assert h.status == 1                              # VSIE_WARN_NOT_CONVERGED, valid handle
    inf = h.info()
    assert max(max(r) for r in inf["ranks"]) <= 4
    assert min(inf["heldout_err"]) > 10 * cfg1.tol


@pytest.mark.parametrize("ci", [2, 4, 3])
def test_heldout_full_size(ci):
    """P27 / T4 on the full-size configs: 1000 seeded held-out indices per chi (PCG64 seed
    12409005, independent of the build's own held-out sample), oracle entries vs TT values.
    cfg 2: values from the exported cores by the oracle's chain product; cfgs 3 / 4 (cores of
    1-6 GB): the device chain product (vsie_coupling_tt_eval), itself checked against the
    oracle's on random cores in test_gpu_apply.py.  cfg 3 is the two-surface body config (the
    r3 ~ 1500 supercores of the Householder-based factorisation)."""
    import torch
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(ci)
    h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1)
    assert h.status == 0
    prob = oent.problem_from_config(cfg)
    s = synth.uniform_indices(tuple(cfg.n) + (cfg.m,), 1000, synth.SEEDS["heldout"])
    v = s[:, 0] + cfg.n[0] * (s[:, 1] + cfg.n[1] * s[:, 2])
    tts = h.export_cores() if ci == 2 else None
    for chi in range(3):
        ref = oent.entries(prob, chi * cfg.n_v + v, s[:, 3])
        if tts is not None:
            got = ttmv.eval_at(tts[chi], s)
        else:
            got = h.tt_eval(torch.from_numpy(chi * cfg.n_v + v), torch.from_numpy(s[:, 3])).cpu().numpy()
        assert validate.rel_l2(got, ref) <= 10 * cfg.tol, (ci, chi)


def test_paper_setting_build_cfg2():
    """The paper's own setting: TT-cross tolerance 1e-3 on the 1 x 1 far rule
    (quad_rule = 1).  Held-out (1000 per chi, seeded) vs the oracle's 1 x 1 entries within
    10 tol; ranks well below the 1e-6 build's (Appendix A probe: (5, 22, 68) at 1e-3)."""
    from paper_2206_12409_b200 import Coupling
    cfg = synth.get_config(2)
    h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, 1e-3, nrhs_max=1, quad_rule=1)
    assert h.status == 0
    inf = h.info()
    assert inf["quad_rule"] == 1 and max(r[2] for r in inf["ranks"]) < 150
    prob = oent.problem_from_config(cfg, quad_rule=1)
    s = synth.uniform_indices(tuple(cfg.n) + (cfg.m,), 1000, synth.SEEDS["heldout"])
    v = s[:, 0] + cfg.n[0] * (s[:, 1] + cfg.n[1] * s[:, 2])
    tts = h.export_cores()
    for chi in range(3):
        ref = oent.entries(prob, chi * cfg.n_v + v, s[:, 3])
        assert validate.rel_l2(ttmv.eval_at(tts[chi], s), ref) <= 1e-2, chi
