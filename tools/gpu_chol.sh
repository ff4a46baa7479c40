# Cholesky probe: event timings at several n
for n in 64 150 200 500 1000 2000; do timeout 120 python tools/chol_bench.py $n; done > gpurun_out/chol_times.log 2>&1
cat gpurun_out/chol_times.log
