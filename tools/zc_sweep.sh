python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for mx in 16 8 4; do VSIE_ZGEMM_CLUSTER_MAX=$mx timeout 300 python tools/pair_timing.py 2 30 > gpurun_out/zc_$mx.json 2>gpurun_out/zc_$mx.err; echo "max $mx rc=$?"; tail -1 gpurun_out/zc_$mx.err; done
VSIE_ZGEMM_CLUSTER=0 timeout 300 python tools/pair_timing.py 2 30 > gpurun_out/zc_off.json 2>&1; echo off rc=$?
