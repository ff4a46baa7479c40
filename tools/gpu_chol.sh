# Cholesky probe: event timings at several n, then one ncu --set full capture of k_chol_df (n=64)
for n in 64 128 256 500 1000 2000; do timeout 120 python tools/chol_bench.py $n; done > gpurun_out/chol_times.log 2>&1
cat gpurun_out/chol_times.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_chol_df --launch-skip 5 -c 1 -o gpurun_out/chol64 python tools/chol_bench.py 64 > gpurun_out/ncu_chol.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_chol.log
