#!/bin/bash
# One GPU call: apply parity tests + pair timing under both G4 schedules + ncu of k_pair_g4.
tag=${1:-pair}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAIL; tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_apply.py -x -q > $out/pytest_apply.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_apply.log
for c in 2 4; do for md in 0 2 3; do
  VSIE_PAIR_G4=$md timeout 300 python tools/pair_timing.py $c 30 > $out/t_cfg${c}_m${md}.json 2> $out/t_cfg${c}_m${md}.err; echo "cfg$c mode$md rc=$?"; cat $out/t_cfg${c}_m${md}.json; tail -2 $out/t_cfg${c}_m${md}.err
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pair_g4 -s 2 -c 1 -o $out/prof python tools/profile_step.py 2 3 > $out/ncu_full.log 2>&1; echo "ncu rc=$?"
