"""GMRES coupling pair steps (vsie_coupling_apply_pair) on cfg cores with the measured ranks
(random values: matvec cost is data independent), for ncu captures.

    python tools/profile_step.py [cfg] [steps] [pair_schedule: auto | g4_shared | g3_shared]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import synth
from paper_2206_12409_b200 import Coupling, grid_of
from gpu_common import rand_tts
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = synth.get_config(ci)
p = os.path.join(ROOT, "profiles", f"ranks_cfg{ci}.json")
ranks = json.load(open(p))["ranks"] if os.path.exists(p) else [cfg.ranks_probe] * 3
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, ranks, 1), nrhs_max=1)
h.configure(graphs=False, pair_schedule=sys.argv[3] if len(sys.argv) > 3 else "auto")
x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
u = torch.from_numpy(synth.complex_gaussian(3 * cfg.n_v, 2)).cuda()
y = torch.empty(3 * cfg.n_v, dtype=torch.complex128, device="cuda")
z = torch.empty(cfg.m, dtype=torch.complex128, device="cuda")
for _ in range(steps):
    h.apply_pair(x, u, "T", out_y=y, out_z=z)
torch.cuda.synchronize()
print("ok", h.info()["apply_launches"] // steps, "launches per step")
