python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/trace.py --rmat-seed 0
