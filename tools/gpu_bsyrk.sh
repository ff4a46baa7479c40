set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -15
CMPC_BATCH_TIMES=1 timeout 300 python tools/batch_lockstep_probe.py 1024 2>&1 | tail -16
timeout 300 ncu --set full --clock-control none -k regex:k_bsyrk -c 1 -o gpurun_out/bsyrk python tools/batch_lockstep_probe.py 256 > gpurun_out/bsyrk_ncu.log 2>&1; tail -3 gpurun_out/bsyrk_ncu.log
