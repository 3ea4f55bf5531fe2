python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_transfer.py tests/test_gpu_parity.py -q -x 2>&1 | tail -15
for c in c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo "$c rc=$?"; tail -3 gpurun_out/b_$c.err; done
python -c "import json; d=json.load(open('gpurun_out/b_c2.json')); print(d['e2e'], d['value'])"
