#!/bin/bash
# One GPU call: ncu launch list + one --set full capture of the pair step of the given configs.
# usage: tools/gpu_ncu_cfg.sh <tag> "<configs>"
tag=${1:-ncu}; cfgs=${2:-3}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
for c in $cfgs; do
  timeout 300 python tools/profile_step.py $c 3 > $out/plain_cfg$c.log 2>&1 || { echo PLAIN FAIL cfg $c; tail $out/plain_cfg$c.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg$c.csv python tools/profile_step.py $c 3 > $out/ncu_launch_cfg$c.log 2>&1; echo "launches cfg $c rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -s 18 -c 18 -o $out/prof_cfg$c python tools/profile_step.py $c 3 > $out/ncu_full_cfg$c.log 2>&1; echo "ncu full cfg $c rc=$?"
  python tools/ncu_summary.py $out/launches_cfg$c.csv $out/prof_cfg$c.ncu-rep $out/ncu_summary_cfg$c.json > /dev/null 2>&1
  rm -f $out/prof_cfg$c.ncu-rep
done
ls $out
