cd $GRAFT_REPO_ROOT
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest -q -x tests/test_gpu_concurrency.py -k lockstep 2>&1 | grep -E "error|Error|passed|failed" | head -5
timeout 300 ncu --set full --clock-control none -k regex:k_b_chol -c 1 -o gpurun_out/bchol2 python tools/batch_lockstep_probe.py 256 > gpurun_out/bchol2.log 2>&1; tail -2 gpurun_out/bchol2.log
