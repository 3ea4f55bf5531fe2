python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_cta.py tests/test_gpu_tail.py tests/test_gpu_report.py tests/test_gpu_errors.py -q -x 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_full.py -q -x -k "c4 or c1 or c3t" 2>&1 | tail -3
timeout 900 python bench.py --config c4 --steps 10 --no-cpu --batch-per-gpu 0 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo "c4 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/b_c4.json')); p=d['paths']; print(p['impl'], p['factor']['us'], p['tail'])"
