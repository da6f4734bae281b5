import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import synth
from oracle import ttmv, validate
from paper_2206_12409_b200 import Coupling, grid_of
from gpu_common import rand_tts
cfg = synth.get_config(1)
for ranks in ([(7,31,73)]*3, [(3,5,7)]*3, [(7,31,73),(7,31,73),(7,30,73)], [(2,3,4)]*3, [(7,20,73)]*3, [(7,31,20)]*3):
    tts = rand_tts(cfg, ranks, 3)
    h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=1)
    x = synth.complex_gaussian(cfg.m, 1)
    y = h.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy().reshape(3, 12*12, 12, order='C')
    yr = ttmv.apply(tts, x, "N").reshape(3, 12*12, 12, order='C')
    y = h.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy().reshape(3, 12, 144)
    yr = ttmv.apply(tts, x, "N").reshape(3, 12, 144)
    err = [validate.rel_l2(y[c, i3], yr[c, i3]) for c in range(3) for i3 in range(12)]
    print(ranks[0], np.array(err).reshape(3, 12).round(3))
