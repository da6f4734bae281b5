"""Entries/s through the C ABI at a config: 1e6 uniform random (row, col) through
vsie_coupling_entries (list mode, the bench's sample) and a structured supercore block of
~2e7 entries through vsie_coupling_supercore (block mode, the cross's shape).

    python tools/entries_rate.py [cfg]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
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
lst = 1e7 / (e0.elapsed_time(e1) * 1e-3)
# block mode: k = 2 supercore with 16 left (i1) and 64 right (n) indices
rng = np.random.default_rng(5)
n1, n2, n3 = cfg.n
left = np.stack([rng.integers(0, n1, 16), np.zeros(16, int)], axis=1)
right = np.stack([rng.integers(0, cfg.m, 64), np.zeros(64, int)], axis=1)
M = h.supercore(1, 2, left, right); torch.cuda.synchronize()
e0.record()
for _ in range(5):
    M = h.supercore(1, 2, left, right)
e1.record(); torch.cuda.synchronize()
blk = 5 * M.numel() / (e0.elapsed_time(e1) * 1e-3)
print(json.dumps({"cfg": ci, "list_entries_per_s": lst, "block_entries_per_s": blk, "block_entries": M.numel(),
                  "pairs_per_s_list": 48 * lst, "pairs_per_s_block": 48 * blk}))
