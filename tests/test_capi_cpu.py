"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and validates arguments / geometry on the host before any
CUDA call (SURVEY §8b error conventions)."""
import ctypes as C

import numpy as np
import pytest

import synth
from paper_2206_12409_b200 import _lib
from paper_2206_12409_b200.coupling import Grid, _meshes_c, _opts


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert "vsie_coupling_build" in syms and "vsie_coupling_apply" in syms and "vsie_coupling_entries" in syms
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) <= set(_lib._SIGS), set(syms) - set(_lib._SIGS)
    assert L.vsie_abi_version() == 4


def test_status_strings_and_defaults():
    L = _lib.lib()
    assert L.vsie_status_string(0) == b"VSIE_OK"
    assert L.vsie_status_string(-2) == b"VSIE_ERR_GEOMETRY"
    assert L.vsie_status_string(1) == b"VSIE_WARN_NOT_CONVERGED"
    o = _lib.vsie_build_opts()
    L.vsie_build_opts_default(C.byref(o))
    assert (o.max_rank, o.max_sweeps, o.oversample, o.heldout, o.world, o.seed) == (2048, 8, 16, 1000, 1, 12409010)
    assert (o.scale_re, o.scale_im) == (1.0, 0.0)
    assert o.quad_rule == 0 and o.test_moment == 0


def _import(grid, meshes, freq=298.2e6, **kw):
    L = _lib.lib()
    g = grid.as_c()
    arr, keep = _meshes_c(meshes)
    o, _ = _opts(**kw)
    ranks = (C.c_int32 * 9)(*([1] * 9))
    dummy = np.zeros(10 ** 6, dtype=np.complex128)
    ptrs = (C.c_void_p * 12)(*([dummy.ctypes.data] * 12))
    h = _lib.HANDLE()
    st = L.vsie_coupling_import_cores(C.byref(g), arr, len(meshes), freq, ranks, ptrs, C.byref(o), C.byref(h))
    return st, h, L.vsie_last_error_message().decode()


def test_argument_errors():
    cfg = synth.get_config(1)
    meshes = cfg.meshes()
    st, h, msg = _import(Grid((0, 12, 12), cfg.h, cfg.origin), meshes)
    assert st == -1 and not h.value and "n must be" in msg
    st, h, msg = _import(Grid(cfg.n, (5e-3, -1.0, 5e-3), cfg.origin), meshes)
    assert st == -1 and not h.value
    st, _, msg = _import(Grid(cfg.n, cfg.h, cfg.origin), meshes, quad_rule=2)
    assert st == -1 and "quad_rule" in msg
    st, h, msg = _import(Grid(cfg.n, cfg.h, cfg.origin), meshes, freq=-1.0)
    assert st == -1 and "freq" in msg
    L = _lib.lib()
    assert L.vsie_coupling_apply(None, None, None, 0, 1, None) == -1
    assert L.vsie_coupling_info(None, None) == -1
    L.vsie_coupling_destroy(None)


def test_geometry_errors():
    cfg = synth.get_config(1)
    grid = Grid(cfg.n, cfg.h, cfg.origin)
    xyz, tri = cfg.meshes()[0]
    bad = tri.copy()
    bad[5] = (bad[5][0], bad[5][0], bad[5][2])          # repeated vertex -> degenerate
    st, _, msg = _import(grid, [(xyz, bad)])
    assert st == -2
    # an edge shared by three triangles (non-manifold)
    extra = np.vstack([tri, [[tri[0][0], tri[0][2], 7]]]).astype(np.int32)
    st, _, msg = _import(grid, [(xyz, extra)])
    assert st == -2 and "more than two" in msg
    # a surface crossing the voxel box violates the non-singular rule
    near = xyz * np.array([0.05, 0.05, 1.0])
    st, _, msg = _import(grid, [(near, tri)])
    assert st == -2 and "10 max(h)" in msg
    # vertex id out of range
    oob = tri.copy()
    oob[0, 0] = len(xyz) + 3
    st, _, _ = _import(grid, [(xyz, oob)])
    assert st == -2


def test_pwl_per_moment_nccl_ids():
    """Each PWL moment handle of a multi-process group gets its own NCCL unique id."""
    import pytest
    from paper_2206_12409_b200 import PWLCoupling
    per = PWLCoupling._per_moment({"world": 2, "rank": 1}, [b"a", b"b", b"c", b"d"])
    assert [p["nccl_unique_id"] for p in per] == [b"a", b"b", b"c", b"d"]
    assert all(p["world"] == 2 and p["rank"] == 1 for p in per)
    assert all("nccl_unique_id" not in p for p in PWLCoupling._per_moment({"world": 1}, None))
    with pytest.raises(ValueError):
        PWLCoupling._per_moment({"nccl_unique_id": b"x"}, None)


def test_farnear_farfar_host_validation():
    """The surface-surface blocks (include/vsie_farnear.h, vsie_farfar.h) reject bad arguments and
    bad meshes on the host, before any CUDA call (runs without a GPU)."""
    L = _lib.lib()
    cfg = synth.get_config(1)
    xyz, tri = cfg.meshes()[0]
    near = synth.near_mesh(1)
    bad = tri.copy()
    bad[3] = (bad[3][1], bad[3][1], bad[3][2])
    o = _lib.vsie_farnear_opts()
    L.vsie_farnear_opts_default(C.byref(o))
    assert (o.max_rank, o.scale_re, o.scale_im, o.device) == (2048, 1.0, 0.0, -1)
    h = _lib.HANDLE()
    an, k1 = _meshes_c([near])
    af, k2 = _meshes_c([(xyz, bad)])
    assert L.vsie_farnear_build(an, 1, af, 1, cfg.freq, 1e-3, C.byref(o), C.byref(h)) == -2 and not h.value
    af, k3 = _meshes_c([(xyz, tri)])
    assert L.vsie_farnear_build(an, 1, af, 1, cfg.freq, 0.0, C.byref(o), C.byref(h)) == -1
    assert L.vsie_farnear_build(an, 1, af, 1, -5.0, 1e-3, C.byref(o), C.byref(h)) == -1
    o.max_rank = 0
    assert L.vsie_farnear_build(an, 1, af, 1, cfg.freq, 1e-3, C.byref(o), C.byref(h)) == -1
    assert L.vsie_farnear_build(None, 0, af, 1, cfg.freq, 1e-3, None, C.byref(h)) == -1
    ab, k4 = _meshes_c([(xyz, bad)])
    assert L.vsie_farfar_build(ab, 1, cfg.freq, 1.0, 0.0, -1, C.byref(h)) == -2
    assert "degenerate" in L.vsie_last_error_message().decode()
    assert L.vsie_farfar_build(af, 1, 0.0, 1.0, 0.0, -1, C.byref(h)) == -1
    assert L.vsie_farfar_build(af, 1, cfg.freq, float("nan"), 0.0, -1, C.byref(h)) == -1
    assert L.vsie_farnear_apply(None, None, None, 0, 1, None) == -1
    assert L.vsie_farfar_apply(None, None, None, 0, 1, 0, None) == -1
    assert L.vsie_farfar_get_info(None, None) == -1
    L.vsie_farnear_destroy(None)
    L.vsie_farfar_destroy(None)
    del k1, k2, k3, k4


def test_set_allocator_arguments():
    """vsie_set_allocator: both hooks or neither (no CUDA call)."""
    L = _lib.lib()
    hook = _lib.ALLOC_FN(lambda n, c: None)
    assert L.vsie_set_allocator(hook, _lib.FREE_FN(), None) == -1
    assert "both" in L.vsie_last_error_message().decode()
    assert L.vsie_set_allocator(_lib.ALLOC_FN(), _lib.FREE_FN(), None) == 0


def test_hybrid_host_validation():
    """vsie_hybrid_*: NULL handles / blocks are rejected on the host (no CUDA call)."""
    L = _lib.lib()
    h = _lib.HANDLE()
    assert L.vsie_hybrid_create(None, None, None, None, None, None, C.byref(h)) == -1
    assert "required" in L.vsie_last_error_message().decode() and not h.value
    assert L.vsie_hybrid_create(None, None, None, None, None, None, None) == -1
    inf = _lib.vsie_gmres_info()
    assert L.vsie_hybrid_gmres(None, None, None, 50, 10, 1e-5, None, C.byref(inf), None) == -1
    assert L.vsie_hybrid_matvec(None, None, None, None) == -1
    hi = _lib.vsie_hybrid_info()
    assert L.vsie_hybrid_get_info(None, C.byref(hi)) == -1
    L.vsie_hybrid_destroy(None)
