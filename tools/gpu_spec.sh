# speculative seg_next: tests, then C2/C3 bench lines and host-turnaround counts
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_speculate.py -x -q > gpurun_out/spec_tests.log 2>&1; echo "spec tests $?"; tail -3 gpurun_out/spec_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests $?"; tail -3 gpurun_out/gpu_tests.log
B="timeout 900 python bench.py"
$B --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/spec_c3.json 2>/dev/null; echo "c3 $?"
$B --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/spec_c2.json 2>/dev/null; echo "c2 $?"
CMPC_GAP_TRACE=1 $B --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep gaps | tail -1
CMPC_GAP_TRACE=1 $B --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep gaps | tail -1
