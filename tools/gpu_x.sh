#!/bin/bash
# One GPU call: A/B of experiment env knobs with tools/pair_timing.py (random cores at the recorded ranks).
# usage: tools/gpu_x.sh <tag> "<configs>" "<env settings, ;-separated>" [reps] ["pytest args" under each env]
tag=${1:-x}; cfgs=${2:-4}; envs=${3:-}; reps=${4:-2}; tests=${5:-}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
IFS=';' read -ra EV <<< "${envs:- }"
for rep in $(seq 1 $reps); do
for e in "${EV[@]}"; do
  for c in $cfgs; do
    n=$(echo "cfg${c}_${e}_$rep" | tr -c 'A-Za-z0-9_\n' '_')
    env $e timeout 300 python tools/pair_timing.py $c 40 > $out/t_$n.json 2> $out/t_$n.err
    echo "== [$e] cfg $c rep $rep rc=$?"; python - "$out/t_$n.json" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
    print(" w", round(d["w"]["ms"], 4), "wr", round(d["wr"]["ms"], 4), "none", round(d["none"]["ms"], 4), d["kernels"])
except Exception as ex:
    print(" FAIL", ex)
PY
  done
done
done
if [ -n "$tests" ]; then
  for e in "${EV[@]}"; do
    env $e timeout 900 python -m pytest $tests -x -q --timeout 600 > $out/pytest_$(echo "$e" | tr -c 'A-Za-z0-9_\n' '_').log 2>&1; echo "pytest [$e] rc=$?"
  done
fi
