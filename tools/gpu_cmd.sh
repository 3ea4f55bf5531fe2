rm -f paper_1812_06160_b200/libjv.so
JV_NVCC_EXTRA=-DJV_HEAVY_PROFILE python -c "import __graft_entry__ as g; g.build()" || exit 1
JV_TRACE=1 timeout 300 python tools/heavy_bench.py 5000 73 > gpurun_out/hb.log 2>&1; grep '"m"' gpurun_out/hb.log
rm -f paper_1812_06160_b200/libjv.so
