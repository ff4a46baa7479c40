# Cholesky check: linalg tests, then timings and the parity tests
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_ipm.py -x -q > gpurun_out/pytest_chol.log 2>&1; echo "linalg/ipm exit $?"; tail -15 gpurun_out/pytest_chol.log
timeout 300 python tools/chol_slope.py
for n in 1000 2000; do timeout 120 python tools/chol_bench.py $n; done
timeout 300 python tools/phases.py ${PHASES:-c5 c3} 2>&1 | grep -E "==|solve:|cholesky|chol_|per-iter"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_par.log 2>&1; echo "parity exit $?"; tail -15 gpurun_out/pytest_par.log
