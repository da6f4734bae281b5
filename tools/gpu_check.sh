#!/bin/bash
# One GPU call during development: build, a pytest selection, optional bench lines.
# usage: tools/gpu_check.sh <tag> "<pytest args>" "<bench configs>"
tag=${1:-chk}; tests=${2:-tests -m gpu}; benches=${3:-}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
if [ -n "$tests" ]; then
  timeout 1800 python -m pytest $tests -x -q --timeout 900 --timeout-method=thread > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
fi
for c in $benches; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_cfg$c.log 2>&1
  echo "bench$c rc=$?"; tail -c 600 $out/bench_cfg$c.log | tail -2
done
