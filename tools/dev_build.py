"""Dev tool: run vsie_coupling_build on a config and check held-out vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import entries as oent, ttmv, validate
from paper_2206_12409_b200 import Coupling, grid_of
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = synth.get_config(ci)
t = time.time()
h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, verbose=int(os.environ.get("VSIE_VERBOSE", "1")), nrhs_max=1, max_sweeps=int(os.environ.get("VSIE_SWEEPS", "8")))
print("build", time.time() - t, "status", h.status)
inf = h.info(); print({k: inf[k] for k in ("ranks", "sweeps", "heldout_err", "entries_evaluated", "build_s", "build_entry_s", "build_factor_s", "build_maxvol_s", "compression")})
tts = h.export_cores()
prob = oent.problem_from_config(cfg)
s = synth.uniform_indices(tuple(cfg.n) + (cfg.m,), 1000, synth.SEEDS["heldout"])
v = s[:, 0] + cfg.n[0] * (s[:, 1] + cfg.n[1] * s[:, 2])
for chi in range(3):
    ref = oent.entries(prob, chi * cfg.n_v + v, s[:, 3])
    print("chi", chi, "heldout oracle", validate.rel_l2(ttmv.eval_at(tts[chi], s), ref))
