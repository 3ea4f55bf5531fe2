"""Race check of the region forward sweep on a random diagonally dominant
matrix: five repeated solves, mismatching rows against the oracle.
(Found the prober / ring-reuse race during development.)"""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from paper_1812_06160_b200 import device as dv, workloads as W, regionplan as RP
a = W.random_diag_dominant(5000, 7, seed=9)
fe = oracle.front_end(a.n, a.row_start, a.col, a.val)
rs, col, diag, val = fe["row_start"], fe["col"], fe["diag"], fe["val"]
n = diag.size
want, bad = oracle.factor_serial(rs, col, val.copy(), diag, 0.0, False)
b = np.random.default_rng(1).uniform(-1, 1, n)
yo = oracle.solve_forward(rs, col, want, b)
d = dv.DevIlu.from_host(n, rs, col, diag, want)
d.region_mode = "on"
rp = d.region_stream("fwd")
print({k: rp[k] for k in ("nreg", "slot_ring", "max_waves", "S", "D", "CS", "CD", "waves", "remote_deps")})
y = dv.empty_f64(n)
for rep in range(5):
    d.solve_async(0, dv.f64(b), y)
    got = dv.host_f64(y, n)
    bad = np.nonzero(got != yo)[0]
    print(rep, "mismatch rows", bad.size, bad[:10])
reg = d.regions()[1]
ws = RP.build_stream("fwd", rs, col, diag, reg, d.regions()[0], 232448 - 2048)
# for the first bad row: its deps and whether remote
if bad.size:
    r = bad[0]
    deps = col[rs[r]:diag[r]]
    print("row", r, "region", reg[r], "deps", deps, "dep regions", reg[deps], "first dep bad?", np.isin(deps, bad))
