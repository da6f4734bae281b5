"""Timeline of one GMRES step (forward + transpose apply) with the chi chains running
concurrently (vsie_coupling_set_timing(h, 2)), plus the graph-replayed step time and the
serialised per-kernel times.  Random cores at the measured ranks (matvec cost is data
independent).

    python tools/trace_step.py [cfg] [steps]
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = synth.get_config(ci)
p = os.path.join(ROOT, "profiles", f"ranks_cfg{ci}.json")
ranks = json.load(open(p))["ranks"] if os.path.exists(p) else [cfg.ranks_probe] * 3
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, ranks, 1), nrhs_max=1)
x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
u = torch.from_numpy(synth.complex_gaussian(3 * cfg.n_v, 2)).cuda()
y = torch.empty(3 * cfg.n_v, dtype=torch.complex128, device="cuda")
z = torch.empty(cfg.m, dtype=torch.complex128, device="cuda")
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
n1, n2, n3 = cfg.n
B = 2 * 16 * (sum(n1 * a + a * n2 * b + b * n3 * c + c * cfg.m for a, b, c in ranks) + cfg.m + 3 * cfg.n_v)


def step():
    h.apply(x, "N", out=y)
    h.apply(u, "T", out=z)


def timed(n, flush_l2=True):
    ts = []
    for i in range(n):
        if flush_l2:
            flush.fill_(i & 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); step(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.mean(ts))


def timed_stream(n, flush_l2):
    """bench.py-style: back-to-back steps on the stream, events per step, one sync."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        if flush_l2:
            flush.fill_(i & 255)
        ev[i][0].record(); step(); ev[i][1].record()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in ev]
    return float(np.median(t)), float(np.mean(t))


for _ in range(5):
    step()
torch.cuda.synchronize()
med, mean = timed(steps)
med_nf, _ = timed(steps, flush_l2=False)
for mode in ("persistent", "batched", "chains"):
    h.configure(mode=mode)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a = timed_stream(steps, True)
    b = timed_stream(steps, False)
    print(json.dumps(dict(mode=mode, stream_flush_ms=a, stream_noflush_ms=b,
                          gbs_flush=B / (a[1] * 1e-3) / 1e9, gbs_noflush=B / (b[1] * 1e-3) / 1e9)))
h.configure(mode="chains")
def step_pair():
    h.apply_pair(x, u, "T", out_y=y, out_z=z)
for _ in range(3):
    step_pair()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for i in range(steps):
    flush.fill_(i & 255)
    ev[i][0].record(); step_pair(); ev[i][1].record()
torch.cuda.synchronize()
tp = float(np.mean([a.elapsed_time(b) for a, b in ev]))
print(json.dumps(dict(mode="pair (apply_pair, chains)", stream_flush_ms=tp, gbs_flush=B / (tp * 1e-3) / 1e9)))
h.configure(mode=os.environ.get('VSIE_MODE', 'chains'))
print(json.dumps(dict(cfg=ci, ranks=ranks, graph_ms_median=med, graph_ms_mean=mean, gbs=B / (mean * 1e-3) / 1e9,
                      graph_ms_median_noflush=med_nf, bytes_per_step=B)))
# serialised per-kernel
h.set_timing(1)
for i in range(steps):
    flush.fill_(i & 255)
    step()
for t in h.timers():
    avg = t["total_ms"] / t["launches"]
    print(f'  serial {t["name"]:16s} {avg*1e3:8.1f} us/launch  x{t["launches"]//steps:2d}/step  '
          f'{t["bytes_per_launch"]/(avg*1e-3)/1e9 if t["bytes_per_launch"] else 0:7.0f} GB/s')
# concurrent timeline (eager)
h.set_timing(2)
for i in range(4):
    flush.fill_(i & 255)
    step()
tr = h.trace()
h.set_timing(0)
last = max(r["call"] for r in tr)
for call in (last - 1, last):
    recs = sorted([r for r in tr if r["call"] == call], key=lambda r: r["t0_ms"])
    print(f"-- call {call} ({'fwd' if call % 2 == 0 else 'adj'}): end {max(r['t1_ms'] for r in recs)*1e3:.1f} us")
    for r in recs:
        print(f'  chi {r["chi"]:2d} {r["name"]:16s} {r["t0_ms"]*1e3:8.1f} -> {r["t1_ms"]*1e3:8.1f} us '
              f'({(r["t1_ms"]-r["t0_ms"])*1e3:6.1f})')
