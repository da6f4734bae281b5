#!/bin/bash
# Round measurement: GPU tests, bench lines (cfg 4 default, 2, 3, 5), the launch list of the
# cfg 4 pair step and one ncu --set full capture of the step's kernels.
# usage: tools/gpu_final.sh <tag> [skip-tests]
tag=${1:-r02}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
python tools/sass_summary.py $out/sass_summary.json > /dev/null 2>&1
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 --timeout-method=thread > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest_gpu.log
fi
timeout 900 python bench.py > $out/bench_cfg4.log 2>&1; echo "bench4 rc=$?"; cp gpurun_out/bench_cfg4_n1.json $out/ 2>/dev/null
timeout 900 python bench.py --config 2 --steps 50 --warmup 5 > $out/bench_cfg2.log 2>&1; echo "bench2 rc=$?"; cp gpurun_out/bench_cfg2_n1.json $out/ 2>/dev/null
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 > $out/bench_cfg3.log 2>&1; echo "bench3 rc=$?"; cp gpurun_out/bench_cfg3_n1.json $out/ 2>/dev/null
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_cfg5.log 2>&1; echo "bench5 rc=$?"; cp gpurun_out/bench_cfg5_n1.json $out/ 2>/dev/null
timeout 300 python tools/profile_step.py 4 3 > $out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/profile_step.py 4 3 > $out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -s 20 -c 20 -o $out/prof python tools/profile_step.py 4 3 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $out/launches.csv $out/prof.ncu-rep $out/ncu_summary.json > /dev/null 2>&1
ls $out
