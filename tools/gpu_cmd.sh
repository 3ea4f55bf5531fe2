python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_errors.py tests/test_gpu_krylov.py -q -x 2>&1 | tail -25 > gpurun_out/t1.txt
timeout 900 python -m pytest tests/test_gpu_full.py -q -x -k "c3t or c4 or c2" 2>&1 | tail -25 >> gpurun_out/t1.txt
cat gpurun_out/t1.txt | tail -40
