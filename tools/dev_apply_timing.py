"""Dev tool: time the TT apply at a config's probe ranks with random cores (no build)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2206_12409_b200 import Coupling, grid_of
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_common import rand_tts

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synth.get_config(ci)
r = cfg.ranks_probe
tts = rand_tts(cfg, [r, r, r], 1)
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
u = torch.from_numpy(synth.complex_gaussian(3 * cfg.n_v, 2)).cuda()
y = torch.empty(3 * cfg.n_v, dtype=torch.complex128, device="cuda")
z = torch.empty(cfg.m, dtype=torch.complex128, device="cuda")
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    h.apply(x, "N", out=y); h.apply(u, "T", out=z)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); h.apply(x, "N", out=y); h.apply(u, "T", out=z); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
h.set_timing(True)
for _ in range(10):
    flush.zero_()
    h.apply(x, "N", out=y); h.apply(u, "T", out=z)
tm = h.timers()
n1, n2, n3 = cfg.n; m = cfg.m
core = 3 * (n1*r[0] + r[0]*n2*r[1] + r[1]*n3*r[2] + r[2]*m)
B = 16 * (core + m + 3*cfg.n_v)
med = float(np.median(ts))
print(json.dumps(dict(cfg=ci, ms_step=med, gbs=2*B/(med*1e-3)/1e9, B_fwd=B)))
for t in tm:
    avg = t["total_ms"]/t["launches"]
    print(f'{t["name"]:22s} {avg*1e3:9.1f} us  {t["bytes_per_launch"]/(avg*1e-3)/1e9 if t["bytes_per_launch"] else 0:8.1f} GB/s  {t["flops_per_launch"]/(avg*1e-3)/1e12 if t["flops_per_launch"] else 0:6.2f} TF')
