#!/bin/bash
# One GPU call: ncu --set full capture of kernels matching a regex in the cfg pair step.
# usage: tools/gpu_ncu.sh <tag> <kernel-regex> [config] [count] [env]
tag=${1:-ncu}; kre=${2:-k_reduce_g1}; cfgi=${3:-4}; cnt=${4:-2}; ev=${5:-}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
env $ev timeout 300 python tools/profile_step.py $cfgi 3 > $out/plain.log 2>&1 || { echo PLAIN FAIL; tail $out/plain.log; exit 1; }
env $ev timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c $cnt -o $out/prof python tools/profile_step.py $cfgi 3 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $out/prof.ncu-rep --page raw --csv > $out/raw.csv 2>/dev/null
ncu -i $out/prof.ncu-rep --page source --csv > $out/source.csv 2>/dev/null
ls -la $out
