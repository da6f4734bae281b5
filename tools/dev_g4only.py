import os, sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch, synth
from paper_2206_12409_b200 import Coupling, grid_of
from gpu_common import rand_tts
cfg = synth.get_config(2)
ranks = json.load(open('/root/repo/profiles/ranks_cfg2.json'))['ranks']
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, ranks, 1), nrhs_max=1)
x = torch.from_numpy(synth.complex_gaussian(cfg.m, 1)).cuda()
y = torch.empty(3 * cfg.n_v, dtype=torch.complex128, device='cuda')
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device='cuda')
for mode in ('persistent', 'batched'):
    h.configure(mode=mode)
    for _ in range(3): h.apply(x, 'N', out=y)
    torch.cuda.synchronize()
    if mode == 'batched':
        h.set_timing(1)
        for i in range(20):
            flush.fill_(i); h.apply(x, 'N', out=y)
        print(mode, [(t['name'], round(t['total_ms']/t['launches']*1e3,1)) for t in h.timers()])
        h.set_timing(0)
    else:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for i in range(20):
            flush.fill_(i); ev[i][0].record(); h.apply(x, 'N', out=y); ev[i][1].record()
        torch.cuda.synchronize()
        print(mode, 'phase-end', os.environ.get('VSIE_MEGA_PHASE_END'), np.mean([a.elapsed_time(b) for a, b in ev]) * 1e3, 'us')
