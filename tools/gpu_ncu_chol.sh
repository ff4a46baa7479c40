# dense-sampled ncu source capture of the standalone dataflow Cholesky (n given)
cd tools/exp
timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:${2:-k_chol_df} --launch-skip 3 -c 1 -o ../../gpurun_out/chol_trace_${1:-64} ./chol_trace ${1:-64} > ../../gpurun_out/ncu_trace.log 2>&1; echo "ncu exit $?"
