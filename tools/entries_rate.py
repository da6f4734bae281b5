"""Entries/s through vsie_coupling_entries: 1e6 uniform random (row, col) at a config
(the bench's entries sample).   python tools/entries_rate.py [cfg]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import synth
from paper_2206_12409_b200 import Coupling, grid_of
from gpu_common import rand_tts

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synth.get_config(ci)
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, [(2, 2, 2)] * 3, 1), nrhs_max=1)
idx = synth.uniform_indices((3 * cfg.n_v, cfg.m), 1_000_000, 424242)
r = torch.from_numpy(idx[:, 0]).cuda(); c = torch.from_numpy(idx[:, 1]).cuda()
h.entries(r, c); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    h.entries(r, c)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"cfg": ci, "entries_per_s": 1e7 / (e0.elapsed_time(e1) * 1e-3), "fast": os.environ.get("VSIE_FAST_SINCOS", "1")}))
