#!/bin/bash
# Round measurement: GPU tests, bench lines (cfg 2 default, 4, 5), launch list and one
# ncu --set full capture of the step's top kernels.  usage: tools/gpu_final.sh <tag>
tag=${1:-r01h}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu.log
timeout 900 python bench.py > $out/bench_cfg2.log 2>&1; echo "bench2 rc=$?"
timeout 900 python bench.py --config 4 --steps 30 --warmup 5 > $out/bench_cfg4.log 2>&1; echo "bench4 rc=$?"
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_cfg5.log 2>&1; echo "bench5 rc=$?"
timeout 300 python tools/profile_step.py 2 3 > $out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/profile_step.py 2 3 > $out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -s 10 -c 13 -o $out/prof python tools/profile_step.py 2 3 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 300 python tools/trace_pair.py 2 > $out/trace2.txt 2>&1
ls $out
