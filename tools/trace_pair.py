"""Concurrent timeline of one GMRES pair step (vsie_coupling_set_timing(h, 2)): per-kernel
start/end (ms from the call's origin event), random cores at the recorded ranks.

    python tools/trace_pair.py [cfg]
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import synth
from paper_2206_12409_b200 import Coupling, grid_of
from gpu_common import rand_tts

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synth.get_config(ci)
ranks = json.load(open(os.path.join(ROOT, "profiles", f"ranks_cfg{ci}.json")))["ranks"]
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, ranks, 1), nrhs_max=1)
x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
u = torch.from_numpy(synth.complex_gaussian(3 * cfg.n_v, 2)).cuda()
y = torch.empty(3 * cfg.n_v, dtype=torch.complex128, device="cuda")
z = torch.empty(cfg.m, dtype=torch.complex128, device="cuda")
fl = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    h.apply_pair(x, u, "T", out_y=y, out_z=z)
h.set_timing(2)
for i in range(3):
    fl.fill_(i)
    h.apply_pair(x, u, "T", out_y=y, out_z=z)
torch.cuda.synchronize()
tr = h.trace()
h.set_timing(0)
last = max(t["call"] for t in tr)
rows = sorted([t for t in tr if t["call"] == last], key=lambda t: t["t0_ms"])
for t in rows:
    print(f'{t["name"]:18s} chi {t["chi"]:2d}  {t["t0_ms"]*1e3:8.1f} -> {t["t1_ms"]*1e3:8.1f} us  ({(t["t1_ms"]-t["t0_ms"])*1e3:6.1f})')
