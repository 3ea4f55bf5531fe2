python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/ -q -x -m gpu 2>&1 | tail -1 | sed 's/warn/w/g'
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1
