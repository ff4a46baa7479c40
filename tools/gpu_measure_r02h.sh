# after the 16-row SYRK shapes: bench lines for configs 2, 3, 4 (T = 50..200), the Markov A/B at
# config 4 and an ncu capture of the config-3 SYRK
set -u
mkdir -p gpurun_out
B="timeout 900 python bench.py"
$B --steps 20 --warmup 5 > gpurun_out/r02h_bench_c3.json 2>/dev/null; echo "c3 $?"
$B --config c2 --steps 20 --warmup 5 > gpurun_out/r02h_bench_c2.json 2>/dev/null; echo "c2 $?"
for T in 50 100 150 200; do $B --config c4 --T $T --steps 5 --warmup 3 > gpurun_out/r02h_bench_c4_T$T.json 2>/dev/null; echo "c4 T=$T $?"; done
timeout 600 python tools/markov_ab.py c4 200 3 | grep -v phases
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_syrk$ --launch-skip 40 -c 1 -o gpurun_out/r02h_syrk python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-markov > gpurun_out/r02h_ncu_syrk.log 2>&1; echo "ncu syrk $?"
