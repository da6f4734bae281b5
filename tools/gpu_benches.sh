#!/bin/bash
# Bench lines for configs 2, 4 and 5 (1 GPU) + an ncu capture of the entry kernel.
out=gpurun_out/benches; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 900 python bench.py --config 2 --steps 30 --warmup 5 > $out/bench2.log 2>&1; echo "bench2 rc=$?"
timeout 900 python bench.py --config 4 --steps 30 --warmup 5 > $out/bench4.log 2>&1; echo "bench4 rc=$?"
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 > $out/bench5.log 2>&1; echo "bench5 rc=$?"
cat > /tmp/ent.py <<'PY'
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch, synth
from gpu_common import grid_of, rand_tts
from paper_2206_12409_b200 import Coupling
cfg = synth.get_config(2)
h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, rand_tts(cfg, [(2, 2, 2)] * 3, 1), nrhs_max=1)
idx = synth.uniform_indices((3 * cfg.n_v, cfg.m), 1_000_000, 424242)
r = torch.from_numpy(idx[:, 0]).cuda(); c = torch.from_numpy(idx[:, 1]).cuda()
for _ in range(3): h.entries(r, c)
torch.cuda.synchronize(); print("ok")
PY
timeout 120 python /tmp/ent.py > $out/ent_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:k_entries_list -s 1 -c 1 -o $out/entries python /tmp/ent.py > $out/ncu_ent.log 2>&1; echo "ncu entries rc=$?"
ls $out
