"""Full TT-cross build of a config on the GPU, then the held-out parity check of
SURVEY §8c-P27 / T4 (1000 seeded indices per chi: oracle entries vs TT values).

    python tools/build_cfg.py <cfg> [max_sweeps]
Writes gpurun_out/build_cfg<cfg>.json and gpurun_out/ranks_cfg<cfg>.json.
"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
from oracle import entries as oent
from oracle import validate
from paper_2206_12409_b200 import Coupling, grid_of

ci = int(sys.argv[1])
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = synth.get_config(ci)
torch.cuda.set_device(0)
t0 = time.perf_counter()
h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1, max_sweeps=sweeps,
                   verbose=int(os.environ.get("VSIE_VERBOSE", "0")))
build_s = time.perf_counter() - t0
inf = h.info()
print("built", ci, "status", h.status, "in", round(build_s, 2), "s; ranks", inf["ranks"], "heldout", inf["heldout_err"],
      "sweeps", inf["sweeps"], flush=True)
prob = oent.problem_from_config(cfg)
s = synth.uniform_indices(tuple(cfg.n) + (cfg.m,), 1000, synth.SEEDS["heldout"])
v = s[:, 0] + cfg.n[0] * (s[:, 1] + cfg.n[1] * s[:, 2])
errs = []
for chi in range(3):
    rows = torch.from_numpy(chi * cfg.n_v + v)
    cols = torch.from_numpy(s[:, 3])
    tt = h.tt_eval(rows, cols).cpu().numpy()
    ref = oent.entries(prob, chi * cfg.n_v + v, s[:, 3])
    errs.append(float(validate.rel_l2(tt, ref)))
print("held-out (oracle entries, PCG64 seed 12409005) rel L2 per chi:", errs, "bound", 10 * cfg.tol, flush=True)
out = dict(cfg=ci, status=h.status, build_s=build_s, ranks=inf["ranks"], heldout_internal=inf["heldout_err"],
           heldout_oracle=errs, bound=10 * cfg.tol, sweeps=inf["sweeps"], entries_evaluated=inf["entries_evaluated"],
           breakdown=dict(entries=inf["build_entry_s"], factor=inf["build_factor_s"], maxvol=inf["build_maxvol_s"]),
           compression=float(inf["compression"]) if inf["compression"] else None,
           core_bytes=inf["core_bytes"])
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"build_cfg{ci}.json"), "w"), indent=1)
json.dump({"ranks": inf["ranks"], "source": "vsie_coupling_build on B200"},
          open(os.path.join(ROOT, "gpurun_out", f"ranks_cfg{ci}.json"), "w"))
