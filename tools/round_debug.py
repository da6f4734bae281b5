"""Diagnostics for vsie_coupling_round on a built config: oracle vs GPU ranks per chi and
the distance of the GPU-rounded TT from its input (test infrastructure: uses oracle/)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))

import synth  # noqa: E402
from oracle import ttmv, ttround  # noqa: E402
from paper_2206_12409_b200 import Coupling, grid_of  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tol = float(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = synth.get_config(ci)
tol = tol if tol is not None else cfg.tol
h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1)
src = h.export_cores()
print("cross ranks", h.info()["ranks"], flush=True)
for chi in range(3):
    t0 = time.perf_counter()
    ref = ttround.tt_round(src[chi], tol)
    print(f"chi {chi}: oracle ranks {ttmv.ranks_of(ref)} ({time.perf_counter() - t0:.1f} s), "
          f"||A|| {ttround.tt_norm(src[chi]):.6e}", flush=True)
t0 = time.perf_counter()
r = h.round(tol)
print("gpu ranks", r, f"{time.perf_counter() - t0:.2f} s", flush=True)
out = h.export_cores()
for chi in range(3):
    nrm = ttround.tt_norm(src[chi])
    print(f"chi {chi}: ||gpu - src|| / ||src|| = {ttround.tt_diff_norm(out[chi], src[chi]) / nrm:.3e}", flush=True)
