python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/ -q -x -m gpu 2>&1 | tail -1 | sed 's/warn/w/g'
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; tail -c 1500 gpurun_out/bench_c2.json
PYTHONPATH=. timeout 300 python tools/rmat_time.py 0 2>&1 | tail -1
