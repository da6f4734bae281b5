#!/bin/bash
# Pair-step timing under environment variants: tools/env_sweep.sh <cfg> "<env1>" "<env2>" ...
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
c=$1; shift
for md in "$@"; do
  tg=$(echo "$md" | tr -d ' =_'); env $md timeout 300 python tools/pair_timing.py $c 30 > gpurun_out/sw_cfg${c}_$tg.json 2> gpurun_out/sw_cfg${c}_$tg.err
  python -c "import json;d=json.load(open('gpurun_out/sw_cfg${c}_$tg.json'));print('$md', round(d['w']['ms']*1e3,1), round(d['none']['ms']*1e3,1))" 2>/dev/null || { echo "$md FAILED"; tail -2 gpurun_out/sw_cfg${c}_$tg.err; }
done
