python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/ -q -x -m gpu 2>&1 | tail -1 | sed 's/warn/w/'
