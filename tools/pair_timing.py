"""Dev tool: time the GMRES coupling pair (vsie_coupling_apply_pair) at a config's recorded
ranks with random cores, under two L2 flush styles, plus the serialised per-kernel times.

    python tools/pair_timing.py [cfg] [steps] [pair_schedule]
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import synth
from paper_2206_12409_b200 import Coupling, grid_of
from gpu_common import rand_tts

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = synth.get_config(ci)
ranks = json.load(open(os.path.join(ROOT, "profiles", f"ranks_cfg{ci}.json")))["ranks"]
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, ranks, 1), nrhs_max=1)
if len(sys.argv) > 3:
    h.configure(pair_schedule=sys.argv[3])
x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
u = torch.from_numpy(synth.complex_gaussian(3 * cfg.n_v, 2)).cuda()
y = torch.empty(3 * cfg.n_v, dtype=torch.complex128, device="cuda")
z = torch.empty(cfg.m, dtype=torch.complex128, device="cuda")
fl = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
fl2 = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
n1, n2, n3 = cfg.n
B = 2 * 16 * (sum(n1 * a + a * n2 * b + b * n3 * c + c * cfg.m for a, b, c in ranks) + cfg.m + 3 * cfg.n_v)


def step():
    h.apply_pair_raw(x.data_ptr(), y.data_ptr(), u.data_ptr(), z.data_ptr(), "T", st)


def flush(style, i):
    fl.fill_(i & 0xFF)
    if style == "wr":
        fl2.sum(dtype=torch.int64)   # read pass: the dirty lines of the write are written back here


out = {"cfg": ci, "ranks": ranks, "schedule": h.info()["pair_schedule"],
       "env": {k: v for k, v in os.environ.items() if k.startswith("VSIE_")}}
for _ in range(5):
    step()
torch.cuda.synchronize()
for style in ("w", "wr", "none"):
    ts = []
    for i in range(steps):
        if style != "none":
            flush(style, i)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); step(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    med = float(np.median(ts))
    out[style] = {"ms": med, "gbs": B / (med * 1e-3) / 1e9}
h.set_timing(True)
for i in range(10):
    flush("w", i)
    step()
torch.cuda.synchronize()
out["kernels"] = {t["name"]: round(1e3 * t["total_ms"] / max(1, t["launches"]), 2) for t in h.timers()}
h.set_timing(False)
print(json.dumps(out))
