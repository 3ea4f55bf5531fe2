python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/ -q -x -m gpu 2>&1 | tail -1 | sed 's/warn/w/'
for c in c1 c2 c3 c4; do timeout 300 python tools/diag.py --config $c > gpurun_out/d.log 2>&1; python -c "import json; d=[json.loads(l) for l in open('gpurun_out/d.log') if l.startswith('{')][-1]; print(d['config'], 'f', round(min(d['factor_ms']),3), 'fw', round(min(d['fwd_ms']),3), 'bw', round(min(d['bwd_ms']),3))"; done
PYTHONPATH=. timeout 300 python tools/rmat_time.py 0 > gpurun_out/r.log 2>&1; tail -1 gpurun_out/r.log
