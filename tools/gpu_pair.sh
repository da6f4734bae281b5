#!/bin/bash
# One GPU call: apply parity tests + pair timing under several schedules + ncu of a kernel.
# usage: tools/gpu_pair.sh <tag> [kernel-regex]
tag=${1:-pair}; kre=${2:-k_seg_gemv}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_apply.py -x -q > $out/pytest_apply.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_apply.log
for c in 2 4; do for md in "VSIE_PAIR_G4=2" "VSIE_PAIR_G4=2 VSIE_REDUCE_TMA=0" "VSIE_PAIR_G4=4"; do
  tg=$(echo $md | tr -d ' =_'); env $md timeout 300 python tools/pair_timing.py $c 30 > $out/t_cfg${c}_$tg.json 2> $out/t_cfg${c}_$tg.err; echo "cfg$c $md rc=$?"; tail -2 $out/t_cfg${c}_$tg.err
done; done
timeout 300 python tools/trace_pair.py 2 > $out/trace2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 1 -c 2 -o $out/prof python tools/profile_step.py 2 3 > $out/ncu_full.log 2>&1; echo "ncu rc=$?"
