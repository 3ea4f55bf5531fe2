python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --config c5 --rmat-count 4 --steps 3 --warmup 3 --cpu-seconds 5 2>&1 | tail -3
