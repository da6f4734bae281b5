#!/bin/bash
# smoke(), the apply GPU tests, and one ncu --set full capture of every kernel of a cfg 2
# pair step (for the dram traffic per launch of profiles/ncu_traffic.json)
out=gpurun_out/traffic; mkdir -p $out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 900 python -m pytest tests/test_gpu_apply.py -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest.log
timeout 300 python tools/profile_step.py 2 2 > $out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -s 13 -c 13 -o $out/prof python tools/profile_step.py 2 2 > $out/ncu.log 2>&1; echo "ncu rc=$?"
