cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -2
CMPC_BATCH_TIMES=1 timeout 300 python tools/batch_lockstep_probe.py 1024 2>&1 | grep -E "syrk|chol|count" | tail -3
