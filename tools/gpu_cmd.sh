python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python tools/trace.py --tridiag 2000
timeout 120 python tools/trace.py --config c2
