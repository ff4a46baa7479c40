# round-2 final measurement set: bench lines per config (with cpu_baseline), a short reference-arm
# check, the C3 launch list and ncu captures of the SYRK and the Cholesky
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
B="timeout 900 python bench.py"
$B --steps 20 --warmup 5 > gpurun_out/r02f_bench_c3.json 2> gpurun_out/r02f_bench_c3.err; echo "c3 $?"
$B --config c1 --steps 20 --warmup 5 > gpurun_out/r02f_bench_c1.json 2>/dev/null; echo "c1 $?"
$B --config c2 --steps 20 --warmup 5 > gpurun_out/r02f_bench_c2.json 2>/dev/null; echo "c2 $?"
for T in 50 100 150 200; do $B --config c4 --T $T --steps 5 --warmup 3 > gpurun_out/r02f_bench_c4_T$T.json 2>/dev/null; echo "c4 T=$T $?"; done
$B --config c5 --steps 5 --warmup 3 > gpurun_out/r02f_bench_c5.json 2>/dev/null; echo "c5 $?"
$B --impl reference --steps 2 --warmup 1 > gpurun_out/r02f_ref_c3.json 2>/dev/null; echo "ref c3 $?"
$B --impl reference --config c5 --steps 3 --warmup 1 > gpurun_out/r02f_ref_c5.json 2>/dev/null; echo "ref c5 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_launch.log 2>&1; echo "launches $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_syrk$ --launch-skip 40 -c 1 -o gpurun_out/r02f_syrk python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_syrk.log 2>&1; echo "ncu syrk $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_chol_df --launch-skip 40 -c 1 -o gpurun_out/r02f_chol python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_chol.log 2>&1; echo "ncu chol $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bsyrk --launch-skip 10 -c 1 -o gpurun_out/r02f_bsyrk python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_bsyrk.log 2>&1; echo "ncu bsyrk $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_b_chol --launch-skip 10 -c 1 -o gpurun_out/r02f_bchol python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_bchol.log 2>&1; echo "ncu bchol $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_launch_c5.log 2>&1; echo "launches c5 $?"
