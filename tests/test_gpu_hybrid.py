"""The GMRES consumer of the hybrid system (include/vsie_hybrid.h) vs the
oracle (oracle/hybrid.py, oracle/gmres.py; pins P52 / P53) on cfg 1 with the near coil of
synth.near_mesh(1).  Every block of the device operator comes from this library's handles;
the oracle composes its own blocks (dense Galerkin matrices, the same TT cores)."""
import numpy as np
import pytest

import synth
from oracle import entries as oent
from oracle import farfar as off
from oracle import farnear as ofn
from oracle import geometry, gmres, hybrid, ttmv, ttsvd, validate

from gpu_common import grid_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def system1(dense1):
    """Oracle blocks of the cfg 1 hybrid system and the device handles built from the same
    definitions (TT cores: oracle TT-SVD imported; Galerkin blocks: built on the device)."""
    import torch
    from paper_2206_12409_b200 import Coupling, FarFar, FarNear, Hybrid
    cfg = synth.get_config(1)
    k0 = 2 * np.pi * cfg.freq / synth.configs.C0
    near = [synth.near_mesh(1)]
    Zff = off.dense_ff(off.rwg_triangle_tables(cfg.meshes()), k0)
    Znn = off.dense_ff(off.rwg_triangle_tables(near), k0)
    rn, jn = geometry.mesh_sources(near)
    rf, jf = geometry.mesh_sources(cfg.meshes())
    Zfn = ofn.dense_cc(rn, jn, rf, jf, k0)
    Dn = oent.dense(oent.make_problem(cfg.n, cfg.h, cfg.origin, near, cfg.freq))
    ttf = [ttsvd.tt_svd(ttmv.tensor_of(dense1, cfg.n, c), cfg.tol) for c in range(3)]
    ttn = [ttsvd.tt_svd(ttmv.tensor_of(Dn, cfg.n, c), cfg.tol) for c in range(3)]
    eps = synth.phantom_eps(cfg.n, cfg.h, cfg.origin, cfg.freq)
    d = hybrid.body_diagonal(cfg.n, cfg.h, eps) * 1e3
    blocks = dict(Zff=Zff, Znn=Znn, Zfn=Zfn, tt_far=ttf, tt_near=ttn, d_body=d)
    dev = dict(
        ff=FarFar.build(cfg.meshes(), cfg.freq),
        nn=FarFar.build(near, cfg.freq),
        fn=FarNear.build(near, cfg.meshes(), cfg.freq, 1e-15),    # every row used: exact U W^T
        cbf=Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, ttf, nrhs_max=1),
        cbn=Coupling.from_cores(grid_of(cfg), near, cfg.freq, ttn, nrhs_max=1),
    )
    d_dev = torch.from_numpy(d).cuda()
    H = Hybrid(dev["ff"], dev["cbf"], d_dev, fn=dev["fn"], nn=dev["nn"], cb_near=dev["cbn"])
    H0 = Hybrid(dev["ff"], dev["cbf"], d_dev)          # no near domain (m_n = 0)
    return cfg, blocks, H, H0, dev


def test_matvec_vs_oracle(system1):
    """The device Eq. 15 operator equals the oracle composition (all blocks, all directions)."""
    import torch
    cfg, blocks, H, H0, dev = system1
    inf = H.info()
    mf, mn = blocks["Zff"].shape[0], blocks["Znn"].shape[0]
    assert (inf["m_far"], inf["m_near"], inf["n_body"], inf["n"]) == (mf, mn, 3 * cfg.n_v, mf + mn + 3 * cfg.n_v)
    assert dev["fn"].info()["rank"] == mn
    for seed in (1, 2):
        x = synth.complex_gaussian(inf["n"], 300 + seed)
        got = H.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        ref = hybrid.matvec(blocks, x)
        assert validate.rel_l2(got, ref) <= 1e-11
        for a, b in ((0, mf), (mf, mf + mn), (mf + mn, inf["n"])):   # every block row
            assert validate.rel_l2(got[a:b], ref[a:b]) <= 1e-10, (a, b)
    # no near domain: Eq. 4 with the far conductors only
    b0 = dict(blocks, Znn=np.zeros((0, 0)), Zfn=np.zeros((0, mf)), tt_near=None)
    x0 = synth.complex_gaussian(mf + 3 * cfg.n_v, 303)
    ref0 = np.concatenate([blocks["Zff"] @ x0[:mf] + ttmv.apply(blocks["tt_far"], x0[mf:], "T"),
                           ttmv.apply(blocks["tt_far"], x0[:mf], "N") + blocks["d_body"] * x0[mf:]])
    got0 = H0.matvec(torch.from_numpy(x0).cuda()).cpu().numpy()
    assert H0.info()["m_near"] == 0 and validate.rel_l2(got0, ref0) <= 1e-11
    del b0


def test_gmres_vs_oracle(system1):
    """Device GMRES follows the oracle's iterates: the same residual history (60 iterations,
    restart 20: three cycles with two restarts) and the same iterate, and its residual
    estimate is the true residual of the returned x."""
    import torch
    cfg, blocks, H, H0, dev = system1
    n = H.info()["n"]
    mf = blocks["Zff"].shape[0]
    b = np.zeros(n, dtype=np.complex128)
    b[:mf] = synth.complex_gaussian(mf, 52)          # voltage excitation on the far conductors
    hist_o = []
    xo, its_o, rel_o = gmres.gmres(lambda v: hybrid.matvec(blocks, v), b, tol=1e-14, restart=20, max_iter=60,
                                   history=hist_o)
    x, info, hist = H.gmres(torch.from_numpy(b).cuda(), restart=20, max_iter=60, tol=1e-14)
    assert info["iterations"] == its_o == 60 and info["restarts"] == 3 and not info["converged"]
    assert np.allclose(hist, hist_o, rtol=1e-6, atol=0), np.max(np.abs(np.array(hist) / hist_o - 1))
    xg = x.cpu().numpy()
    assert validate.rel_l2(xg, xo) <= 1e-6
    true = np.linalg.norm(hybrid.matvec(blocks, xg) - b) / np.linalg.norm(b)
    assert abs(true - info["rel_residual"]) <= 1e-6 * true
    # the paper's setting: tol 1e-5, restart 50 -- a stopping run returns a converged iterate
    # on the well-conditioned body-only part (far rows scaled out: b on the body unknowns)
    bb = np.zeros(n, dtype=np.complex128)
    bb[-3 * cfg.n_v:] = synth.complex_gaussian(3 * cfg.n_v, 53)
    xb, ib, hb = H.gmres(torch.from_numpy(bb).cuda(), restart=50, max_iter=400, tol=1e-5)
    hist_b = []
    _, its_b, _ = gmres.gmres(lambda v: hybrid.matvec(blocks, v), bb, tol=1e-5, restart=50, max_iter=400,
                              history=hist_b)
    assert ib["iterations"] == its_b and (ib["converged"] == (hist_b[-1] <= 1e-5))
    if ib["converged"]:
        tb = np.linalg.norm(hybrid.matvec(blocks, xb.cpu().numpy()) - bb) / np.linalg.norm(bb)
        assert tb <= 1.5e-5


def test_gmres_edge_cases(system1):
    import torch
    from paper_2206_12409_b200 import VsieError
    cfg, blocks, H, H0, dev = system1
    n = H.info()["n"]
    z = torch.zeros(n, dtype=torch.complex128, device="cuda")
    x, info, hist = H.gmres(z, restart=5, max_iter=10)
    assert info["iterations"] == 0 and info["converged"] and not torch.any(x)
    with pytest.raises(VsieError):
        H.gmres(z, restart=0)
    with pytest.raises(VsieError):
        H.gmres(z, tol=0.0)


def test_matvec_full_size_composition():
    """cfg 4 (N = 31.7 M unknowns): the hybrid operator equals the composition of its block
    handles' own applies (each parity-tested against the oracle in its own test file), block
    row by block row -- offsets, strides and 64-bit indexing of the staged matvec at scale --
    and a few GMRES iterations keep the recurrence residual equal to the true residual."""
    import torch
    from gpu_common import rand_tts
    from paper_2206_12409_b200 import Coupling, FarFar, FarNear, Hybrid
    cfg = synth.get_config(4)
    near = [synth.near_mesh(4)]
    ff = FarFar.build(cfg.meshes(), cfg.freq)
    nn = FarFar.build(near, cfg.freq)
    fn = FarNear.build(near, cfg.meshes(), cfg.freq, 1e-3)
    mf, mn = ff.info()["m"], nn.info()["m"]
    cbf = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, [(3, 5, 7)] * 3, 61), nrhs_max=1)
    ttn = [[c for c in tt] for tt in rand_tts(cfg, [(2, 4, 6)] * 3, 62)]
    dims_n = tuple(cfg.n) + (mn,)
    rng = np.random.default_rng(63)
    for tt in ttn:   # the near coupling's last mode has m_n columns
        r3 = tt[3].shape[0]
        tt[3] = (rng.normal(size=(r3, dims_n[3], 1)) + 1j * rng.normal(size=(r3, dims_n[3], 1))) / np.sqrt(2 * r3)
    cbn = Coupling.from_cores(grid_of(cfg), near, cfg.freq, ttn, nrhs_max=1)
    nb = 3 * cfg.n_v
    d = torch.from_numpy(synth.complex_gaussian(nb, 64)).cuda()
    H = Hybrid(ff, cbf, d, fn=fn, nn=nn, cb_near=cbn)
    n = H.info()["n"]
    assert n == mf + mn + nb
    x = torch.from_numpy(synth.complex_gaussian(n, 65)).cuda()
    y = H.matvec(x)
    xf, xn, xb = x[:mf], x[mf:mf + mn], x[mf + mn:]
    yb_c, zf_c = cbf.apply_pair(xf, xb, "T")
    yb_n, zn_c = cbn.apply_pair(xn, xb, "T")
    yn_fn, yf_fn = fn.apply_pair(xf, xn)
    ref_f = ff.apply(xf) + zf_c + yf_fn
    ref_n = nn.apply(xn) + zn_c + yn_fn
    ref_b = yb_c + yb_n + d * xb
    for got, ref in ((y[:mf], ref_f), (y[mf:mf + mn], ref_n), (y[mf + mn:], ref_b)):
        assert ((got - ref).norm() / ref.norm()).item() <= 1e-13
    b = torch.zeros(n, dtype=torch.complex128, device="cuda")
    b[:mf] = xf
    xs, info, hist = H.gmres(b, restart=3, max_iter=4, tol=1e-30)
    assert info["iterations"] == 4 and info["restarts"] == 2
    true = ((H.matvec(xs) - b).norm() / b.norm()).item()
    assert abs(true - info["rel_residual"]) <= 1e-6 * true
