# round-2 last build (speculative segment, Markov table): bench lines per config and the C3 / C5
# launch lists (the kernel captures of r02f stand; the Markov-path captures are r02g_ncu_full_markov)
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
B="timeout 900 python bench.py"
$B --steps 20 --warmup 5 > gpurun_out/r02g_bench_c3.json 2> gpurun_out/r02g_bench_c3.err; echo "c3 $?"
$B --config c1 --steps 20 --warmup 5 > gpurun_out/r02g_bench_c1.json 2>/dev/null; echo "c1 $?"
$B --config c2 --steps 20 --warmup 5 > gpurun_out/r02g_bench_c2.json 2>/dev/null; echo "c2 $?"
for T in 50 100 150 200; do $B --config c4 --T $T --steps 5 --warmup 3 > gpurun_out/r02g_bench_c4_T$T.json 2>/dev/null; echo "c4 T=$T $?"; done
$B --config c5 --steps 5 --warmup 3 > gpurun_out/r02g_bench_c5.json 2>/dev/null; echo "c5 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02g_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-markov > gpurun_out/r02g_ncu_launch.log 2>&1; echo "launches $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02g_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-markov > gpurun_out/r02g_ncu_launch_c5.log 2>&1; echo "launches c5 $?"
