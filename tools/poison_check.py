"""Dev check: TT-cross build of a config on ordinary buffers vs buffers pre-filled with a byte
pattern through the allocation hook (finds reads of never-written device memory).

    python tools/poison_check.py [cfg] [byte ...]"""
import ctypes, glob, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import synth
from paper_2206_12409_b200 import Coupling, grid_of, set_allocator

rt = None
for c in glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*")):
    rt = ctypes.CDLL(c)
rt.cudaMemset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
pats = [int(b, 0) for b in sys.argv[2:]] or [0xFF, 0x00]
cfg = synth.get_config(ci)


def build(pat):
    if pat is not None:
        def _alloc(n):
            p = torch.cuda.caching_allocator_alloc(int(n))
            rt.cudaMemset(p, pat, int(n))
            return p
        set_allocator(_alloc, torch.cuda.caching_allocator_delete)
    try:
        h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1, verbose=1)
    finally:
        set_allocator(None, None)
    return h


h0 = build(None)
c0 = h0.export_cores()
i0 = h0.info()
print("normal", i0["ranks"], i0["heldout_err"], i0["sweeps"], flush=True)
for pat in pats:
    h = build(pat)
    i = h.info()
    c = h.export_cores()
    d = [[float(np.max(np.abs(c0[x][k] - c[x][k]))) if c0[x][k].shape == c[x][k].shape else "shape"
          for k in range(4)] for x in range(3)]
    print(hex(pat), i["ranks"], i["heldout_err"], i["sweeps"], "core diffs", d, flush=True)
