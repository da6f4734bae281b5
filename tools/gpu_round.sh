#!/bin/bash
# One GPU call: parity tests, bench line, launch list and one ncu --set full capture.
# usage: tools/gpu_round.sh <tag> [kernel-regex] [config]
tag=${1:-r01}; kre=${2:-k_gemv_n}; cfgi=${3:-2}
out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
timeout 900 python bench.py --config $cfgi --steps 30 --warmup 5 > $out/bench.log 2>&1; echo "bench rc=$?"; tail -c 400 $out/bench.log
timeout 300 python tools/profile_step.py $cfgi 3 > $out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/profile_step.py $cfgi 3 > $out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 3 -o $out/prof python tools/profile_step.py $cfgi 3 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls $out
