"""Per-tile timeline of the persistent apply (vsie_coupling_set_tile_trace): for each
(phase, chi) segment the tile count, first start / last end and mean tile time, plus
the busy fraction of the CTAs over the launch.

    python tools/tile_trace.py [cfg] [order]
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
cfg = synth.get_config(ci)
p = os.path.join(ROOT, "profiles", f"ranks_cfg{ci}.json")
ranks = json.load(open(p))["ranks"] if os.path.exists(p) else [cfg.ranks_probe] * 3
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, ranks, 1), nrhs_max=1)
h.configure(persistent=True)
x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
u = torch.from_numpy(synth.complex_gaussian(3 * cfg.n_v, 2)).cuda()
y = torch.empty(3 * cfg.n_v, dtype=torch.complex128, device="cuda")
z = torch.empty(cfg.m, dtype=torch.complex128, device="cuda")
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
names = {0: ["G4 x", "G3 y4", "G2 Y3", "G1 Y2"], 1: ["G1^T u", "G2^T W1", "G3^T W2", "G4^T z3 + sum"]}
for _ in range(3):
    h.apply(x, "N", out=y); h.apply(u, "T", out=z)
h.set_tile_trace(True)
for d, (v, o, op) in enumerate(((x, y, "N"), (u, z, "T"))):
    for _ in range(2):
        flush.fill_(1)
        h.apply(v, op, out=o)
    torch.cuda.synchronize()
    recs = h.tile_trace(d)
    end = max(r["t1_us"] for r in recs)
    print(f"== direction {'fwd' if d == 0 else 'adj'}: {len(recs)} tiles, span {end:.1f} us")
    seg = {}
    for r in recs:
        seg.setdefault((r["phase"], r["chi"]), []).append(r)
    for (ph, c), rs in sorted(seg.items(), key=lambda kv: min(r["t0_us"] for r in kv[1])):
        t0 = min(r["t0_us"] for r in rs); t1 = max(r["t1_us"] for r in rs)
        dur = np.array([r["t1_us"] - r["ready_us"] for r in rs])
        wt = np.array([r["ready_us"] - r["t0_us"] for r in rs])
        print(f"  ph {ph} {names[d][ph]:14s} chi {c}: {len(rs):4d} tiles  {t0:7.1f} -> {t1:7.1f} us  "
              f"work mean {dur.mean():6.1f} max {dur.max():6.1f} us, wait mean {wt.mean():6.1f} max {wt.max():6.1f}")
    by_sm = {}
    for r in recs:
        by_sm.setdefault(r["sm"], []).append(r["t1_us"] - r["ready_us"])
    busy = sum(sum(v) for v in by_sm.values())
    waits = sum(r["ready_us"] - r["t0_us"] for r in recs)
    print(f"  SMs used {len(by_sm)}, working tile-time / (SMs x span) = {busy / (len(by_sm) * end):.2f}, "
          f"waiting {waits / (len(by_sm) * end):.2f} (2 CTAs per SM -> max 2.0)")
h.set_tile_trace(False)
