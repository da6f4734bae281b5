#!/bin/bash
out=gpurun_out/prof2; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || exit 1
timeout 300 python tools/trace_pair.py 2 > $out/trace2.txt 2>&1; echo trace rc=$?
timeout 300 python tools/trace_pair.py 4 > $out/trace4.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_reduce_g1|k_expand_g1|k_zgemm_tc|k_gemv_t|k_gemv_n_cp|k_splitk" -s 20 -c 8 -o $out/prof python tools/profile_step.py 2 3 > $out/ncu_full.log 2>&1; echo "ncu rc=$?"
