python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --steps 3 --warmup 3 --no-cpu"
$B > gpurun_out/plain_bench.json 2> gpurun_out/plain_bench.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"factor_kernel|solve_kernel|spmv_stream" -s 12 -c 4 -o gpurun_out/prof_r01_c2 $B > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
