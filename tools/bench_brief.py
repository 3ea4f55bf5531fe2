"""One-screen summary of a bench.py JSON line: python tools/bench_brief.py FILE"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value %.4g %s  step %.4f ms  parity %s  impl %s" % (
    d["value"], d["unit"], d["ms_per_step"], d.get("parity_vs_reference"), d["paths"]["impl"]))
e = d.get("e2e", {})
print("e2e %.4g ms %.3f" % (e.get("value", 0), e.get("ms", 0)), e.get("precond_lambda"))
for k, v in d["rooflines"].items():
    print("  %-7s %9.1f us  frac %.4f  %s" % (k, v["us"], v["frac"], v["kernel"]))
print("  clocks", d.get("clocks"))
