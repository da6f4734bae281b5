"""GPU dense far-far block (include/vsie_farfar.h) vs oracle/farfar.py.

Entries: the stored tiles (cfg 1, the whole 1128 x 1128 matrix) and the list kernel (sampled at
cfg 2 / cfg 4 sizes, near pairs included) against the oracle element by element, scale-relative
1e-12 (the §8c-T1 bar; the analytic potentials add logs / atans, both sides in FP64).  Apply:
against the dense oracle product (cfg 1) and, at full size (cfg 4: 39890 RWG, 12.8 GB of tiles),
on sampled output rows computed from oracle entries one by one.
"""
import numpy as np
import pytest

import synth
from oracle import farfar as off

pytestmark = pytest.mark.gpu


def _tables(ci):
    cfg = synth.get_config(ci)
    return cfg, off.rwg_triangle_tables(cfg.meshes()), 2 * np.pi * cfg.freq / synth.configs.C0


@pytest.fixture(scope="module")
def dense1():
    cfg, T, k0 = _tables(1)
    return off.dense_ff(T, k0)


def test_tiles_cfg1_equal_oracle_dense(dense1):
    from paper_2206_12409_b200 import FarFar
    cfg = synth.get_config(1)
    h = FarFar.build(cfg.meshes(), cfg.freq)
    inf = h.info()
    assert inf["m"] == 1128 and inf["tiles"] == 9 * 10 // 2 and inf["near_pairs"] > 0
    Z = h.export()
    assert np.max(np.abs(Z - dense1)) <= 1e-12 * np.max(np.abs(dense1))
    assert np.array_equal(Z, Z.T)
    # list kernel == tiles (same entry function)
    rng = np.random.default_rng(60)
    r = rng.integers(0, 1128, 3000)
    c = rng.integers(0, 1128, 3000)
    got = h.entries(r, c).cpu().numpy()
    assert np.array_equal(got, Z[r, c])


def test_apply_ops_cfg1(dense1):
    import torch
    from paper_2206_12409_b200 import FarFar
    cfg = synth.get_config(1)
    h = FarFar.build(cfg.meshes(), cfg.freq, scale=2.0 - 0.5j)
    Zs = (2.0 - 0.5j) * dense1
    for op, ref_m in (("N", Zs), ("T", Zs.T), ("C", Zs.conj().T)):
        for nrhs in (1, 2):
            x = synth.complex_gaussian(1128 * nrhs, 6100 + nrhs).reshape(1128, nrhs, order="F")
            xx = x[:, 0] if nrhs == 1 else x
            got = h.apply(torch.from_numpy(xx).cuda(), op).cpu().numpy()
            ref = ref_m @ xx
            assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)), (op, nrhs)
    # accumulate: y += Z x
    x = torch.from_numpy(synth.complex_gaussian(1128, 6110)).cuda()
    y0 = torch.from_numpy(synth.complex_gaussian(1128, 6111)).cuda()
    y = y0.clone()
    h.apply(x, "N", out=y, accumulate=True)
    assert torch.allclose(y, y0 + h.apply(x, "N"), rtol=0, atol=1e-13 * float(y.abs().max()))


@pytest.mark.parametrize("ci", [2, 4])
def test_entries_and_apply_full_size(ci):
    """Sampled entries (uniform + the diagonal + near neighbours) and sampled rows of y = Z x at
    the full far-surface size of the config."""
    import torch
    from paper_2206_12409_b200 import FarFar
    cfg, T, k0 = _tables(ci)
    m = len(T["l"])
    h = FarFar.build(cfg.meshes(), cfg.freq)
    inf = h.info()
    assert inf["m"] == m and inf["matrix_bytes"] == 16 * 128 * 128 * inf["tiles"]
    rng = np.random.default_rng(62 + ci)
    r = np.concatenate([rng.integers(0, m, 4000), np.arange(0, m, 97), np.arange(1, m, 131)])
    c = np.concatenate([rng.integers(0, m, 4000), np.arange(0, m, 97), np.arange(0, m - 1, 131)])
    got = h.entries(r, c).cpu().numpy()
    ref = off.entries_ff(T, k0, r, c)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    x = synth.complex_gaussian(m, 6200 + ci)
    y = h.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy()
    for row in (0, m // 3, m - 1):
        zr = off.entries_ff(T, k0, np.full(m, row), np.arange(m))
        yr = zr @ x
        assert abs(y[row] - yr) <= 1e-11 * np.sum(np.abs(zr) * np.abs(x)), (row, y[row], yr)
