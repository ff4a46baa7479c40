# SYRK iteration: linalg + structure GPU tests, full GPU suite, per-phase timings with the plan stats
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -m pytest tests/test_gpu_linalg.py -x -q > gpurun_out/pytest_linalg.log 2>&1; echo "linalg exit $?"; tail -3 gpurun_out/pytest_linalg.log
CMPC_SYRK_PLAN=1 timeout 300 python tools/phases.py ${PHASES:-c2 c3 c4 c5} > gpurun_out/phases.log 2>&1; echo "phases exit $?"
grep -v "^ *$" gpurun_out/phases.log | grep -E "==|syrk plan|condense|solve:|per-iter"
if [ -n "$FULLTESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log; fi
