#!/bin/bash
# Cross / round GPU tests, then verbose TT-cross builds with the oracle held-out check.
# usage: tools/gpu_build_check.sh <tag> "<configs>"
tag=${1:-bld}; cfgs=${2:-"2 4"}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_cross.py tests/test_gpu_round.py -x -q --timeout 600 --timeout-method=thread > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
for c in $cfgs; do
  VSIE_VERBOSE=1 timeout 1500 python tools/build_cfg.py $c > $out/build_cfg$c.log 2>&1; echo "build cfg$c rc=$?"; grep -E "^built|held-out" $out/build_cfg$c.log
done
