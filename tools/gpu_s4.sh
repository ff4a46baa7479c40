nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?"
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo "bench c4 exit $?"
timeout 900 python bench.py --config c5 > gpurun_out/bench_c5.log 2>&1; echo "bench c5 exit $?"
timeout 300 python tools/phases.py c2 c3 c4 c5 > gpurun_out/phases.log 2>&1; echo "phases exit $?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/prof_c3.py > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/build_launches.csv python tools/build_only.py > gpurun_out/bo.log 2>&1; echo "ncu build exit $?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:'^(k_syrk|k_chol_df|k_proto_gemv|k_syrk_reduce|k_jtpl_symv|k_res_rows|k_proto_reduce)$' --launch-skip 24 -c 8 -o gpurun_out/full_c3 python tools/prof_c3.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
