# round-2 GPU call: the GPU test suite (all failures listed), then a short C3 bench
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nproc; grep -m1 "model name" /proc/cpuinfo
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest_gpu.log
if [ -n "${BENCH:-1}" ]; then
  timeout 600 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench exit $?"
  tail -c 3000 gpurun_out/bench.log
fi
