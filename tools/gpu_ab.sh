#!/bin/bash
# One GPU call during kernel work: build, a pytest selection, traces and bench lines under env A/B.
# usage: tools/gpu_ab.sh <tag> "<pytest args or empty>" "<configs>" "<env settings, ;-separated>"
tag=${1:-ab}; tests=${2:-}; cfgs=${3:-4}; envs=${4:-}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
if [ -n "$tests" ]; then
  timeout 1500 python -m pytest $tests -x -q --timeout 900 > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
fi
IFS=';' read -ra EV <<< "${envs:- }"
for e in "${EV[@]}"; do
  for c in $cfgs; do
    n=$(echo "cfg${c}_$e" | tr -c 'A-Za-z0-9_\n' '_')
    env $e timeout 300 python tools/trace_pair.py $c > $out/trace_$n.txt 2>&1
    env $e timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_$n.log 2>&1
    echo "== $e cfg $c rc=$?"; python - "$out/bench_$n.log" <<'PY'
import json, sys
ls = [l for l in open(sys.argv[1]) if l.startswith("{")]
if ls:
    d = json.loads(ls[-1]); r = d.get("roofline", {})
    print(" ms", round(d["ms_per_step"], 4), "moved_gbs", round(d["config"].get("moved_gbs", 0)), "step_frac", round(r.get("step_frac", 0), 3),
          "dom", r.get("kernel"), round(r.get("avg_us", 0), 1), "us frac", round(r.get("frac", 0), 3))
PY
  done
done
