set -x
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -5
CMPC_BATCH_TIMES=1 timeout 300 python tools/batch_lockstep_probe.py 1024 2>&1 | tail -30
cd tools/exp && timeout 120 ./f32_bench 5 2>&1 | tail -30
