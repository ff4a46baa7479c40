# round measurement: GPU tests, bench, launch list, one ncu --set full capture of the top kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench.log
timeout 300 python tools/phases.py c2 c3 c4 c5 > gpurun_out/phases.log 2>&1; echo "phases exit $?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/prof_c3.py > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
python tools/ncu_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -16 gpurun_out/launches_summary.txt
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:'^(k_syrk|k_chol_df|k_proto_gemv|k_ptq_partial|k_syrk_reduce)$' --launch-skip 24 -c 6 -o gpurun_out/full_c3 python tools/prof_c3.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
