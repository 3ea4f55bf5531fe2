rm -f paper_1812_06160_b200/libjv.so
JV_NVCC_EXTRA=-DJV_HEAVY_PROFILE python -c "import __graft_entry__ as g; g.build()" || exit 1
for a in "5000 73" "5000 8" "5000 1"; do JV_TRACE=1 timeout 300 python tools/heavy_bench.py $a 2>&1 | tail -1; done
rm -f paper_1812_06160_b200/libjv.so
