# ncu --set full of the spmv kernels on c2 (stream kernel and the persistent bulk kernel)
for impl in ${IMPLS:-1}; do
  JV_SPMV_IMPL=$impl JV_SPMV_CFG=${JV_SPMV_CFG:-0} ncu --set full --clock-control none --import-source on \
    -k regex:spmv_ -s 3 -c 1 -o gpurun_out/spmv_impl$impl -f python tools/spmv_bench.py c2 5 > gpurun_out/spmv_ncu$impl.log 2>&1
  tail -2 gpurun_out/spmv_ncu$impl.log
done
