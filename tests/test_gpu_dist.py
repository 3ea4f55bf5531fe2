"""GPU side of the sharded spmv: every rank's plan is run in one process on
cuda:0 through the libjv kernels (jv_gather packs, jv_spmv_rows for the
interior / boundary halves); the NCCL transfer is emulated by device copies
between the ranks' buffers.  Bitwise against the pinned oracle."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")
from paper_1812_06160_b200 import dist as jd  # noqa: E402
from paper_1812_06160_b200 import device as dv  # noqa: E402
from paper_1812_06160_b200 import workloads as W  # noqa: E402


@pytest.mark.parametrize("parts", [2, 3, 8])
@pytest.mark.parametrize("name", ["laplace7", "rmat", "convdiff3d"])
def test_sharded_spmv_on_device(name, parts):
    a = {"laplace7": lambda: W.laplace7(20), "rmat": lambda: W.rmat(12, 5),
         "convdiff3d": lambda: W.convdiff3d(16)}[name]()
    x = np.random.default_rng(9).uniform(-1, 1, a.n)
    want = oracle.spmv(a.row_start, a.col, a.val, x)
    plans = jd.plan_halo_all(a.row_start, a.col, parts, a.val)
    sps = [jd.DistSpmv(p, jd.DeviceOps()) for p in plans]
    xd = dv.f64(x)
    ys = []
    for sp in sps:
        sp.x_local.copy_(xd[sp.plan.lo:sp.plan.hi])
        sp.pack()
    for sp in sps:
        for q, off, m in sp.plan.recv:
            buf = [s for s in sps[q].send if s[0] == sp.plan.rank][0][3]
            sp.x_ext[off:off + m].copy_(buf[:m])
    for sp in sps:
        y = dv.empty_f64(max(sp.plan.n_local, 1))
        sp.interior(y)
        sp.boundary(y)
        ys.append(dv.host_f64(y, sp.plan.n_local))
    got = np.concatenate(ys)
    assert np.array_equal(got, want)   # hub rows included (serial chunked sum)
