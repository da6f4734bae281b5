"""The device-allocation hook (vsie_set_allocator): a handle whose buffers
come from PyTorch's caching allocator gives the same applies as a cudaMalloc handle, its
memory shows up in torch's accounting while it lives and is returned on destroy."""
import numpy as np
import pytest

import synth
from oracle import ttmv, validate

from gpu_common import grid_of, rand_tts

pytestmark = pytest.mark.gpu


def test_torch_allocator_hook():
    import torch
    from paper_2206_12409_b200 import Coupling, use_torch_allocator
    cfg = synth.get_config(2)
    tts = rand_tts(cfg, [(10, 71, 270), (10, 71, 271), (9, 64, 262)], 77)
    x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
    u = torch.from_numpy(synth.complex_gaussian(3 * cfg.n_v, 2)).cuda()
    h0 = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    y0, z0 = h0.apply(x, "N"), h0.apply(u, "T")
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    use_torch_allocator(True)
    try:
        h1 = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
        held = torch.cuda.memory_allocated() - before
        assert held >= h1.info()["core_bytes"], (held, h1.info()["core_bytes"])
        y1, z1 = h1.apply(x, "N"), h1.apply(u, "T")
        yp, zp = torch.empty_like(y1), torch.empty_like(z1)
        h1.apply_pair(x, u, "T", out_y=yp, out_z=zp)
        assert torch.equal(y1, y0) and torch.equal(z1, z0)
        assert torch.equal(yp, y0) and torch.equal(zp, z0)
        h1.close()
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated() - before < held
    finally:
        use_torch_allocator(False)
    # back on cudaMalloc: a new handle does not touch torch's pool
    mid = torch.cuda.memory_allocated()
    h2 = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    assert torch.cuda.memory_allocated() == mid
    xs = synth.complex_gaussian(cfg.m, 1)
    assert validate.rel_l2(h2.apply(torch.from_numpy(xs).cuda(), "N").cpu().numpy(),
                           ttmv.apply(tts, xs, "N")) <= 1e-12


def _cudart():
    import ctypes
    import glob
    import os
    import torch
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                   "libcudart.so*")) + ["/usr/local/cuda/lib64/libcudart.so"]
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError:
            continue
    pytest.skip("no libcudart to poison allocations with")


def test_poisoned_allocations_do_not_change_results():
    """An initcheck substitute (compute-sanitizer is closed on this pool): every library buffer
    starts filled with 0xFF bytes (a NaN pattern) through the allocation hook.  A kernel that
    read memory nobody wrote would turn results into NaN or change them; the cfg 1 TT-cross
    build (cores, ranks, held-out) and cfg 2 applies / pair must be bitwise identical to the
    ones on ordinary cudaMalloc buffers."""
    import ctypes
    import torch
    from paper_2206_12409_b200 import Coupling, set_allocator
    rt = _cudart()
    rt.cudaMemset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]

    def poisoned(enable):
        if not enable:
            set_allocator(None, None)
            return

        def _alloc(n):
            p = torch.cuda.caching_allocator_alloc(int(n))
            assert rt.cudaMemset(p, 0xFF, int(n)) == 0
            return p
        set_allocator(_alloc, torch.cuda.caching_allocator_delete)

    cfg = synth.get_config(1)
    b0 = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=4)
    poisoned(True)
    try:
        b1 = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=4)
    finally:
        poisoned(False)
    i0, i1 = b0.info(), b1.info()
    assert i0["ranks"] == i1["ranks"] and i0["heldout_err"] == i1["heldout_err"]
    for a, b in zip(b0.export_cores(), b1.export_cores()):
        for ca, cb in zip(a, b):
            assert np.array_equal(ca, cb)
    c2 = synth.get_config(2)
    tts = rand_tts(c2, [(10, 71, 270), (10, 71, 271), (9, 64, 262)], 78)
    x = torch.from_numpy(synth.complex_gaussian(c2.m, 1)).cuda()
    u = torch.from_numpy(synth.complex_gaussian(3 * c2.n_v, 2)).cuda()
    outs = []
    for poison in (False, True):
        poisoned(poison)
        try:
            h = Coupling.from_cores(grid_of(c2), c2.meshes(), c2.freq, tts, nrhs_max=4)
            y, z = torch.empty_like(u), torch.empty_like(x)
            h.apply_pair(x, u, "C", out_y=y, out_z=z)
            X = torch.from_numpy(synth.complex_gaussian(c2.m, 3, ncols=4)).cuda()
            outs.append((h.apply(x, "N"), h.apply(u, "T"), y, z, h.apply(X, "N")))
            torch.cuda.synchronize()
            h.close()
        finally:
            poisoned(False)
    for a, b in zip(*outs):
        assert not torch.isnan(b).any() and torch.equal(a, b)
