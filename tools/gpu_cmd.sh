python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -q -x 2>&1 | tail -2
timeout 300 python tools/region_test.py c1 2>&1 | grep -E "cycles|\"parts\""
timeout 300 python tools/region_test.py c2 2>&1 | grep -E "cycles|\"parts\""
