"""Device RCM (jv_rcm_device) equals the host C++ RCM (jv_rcm_host), which is
pinned to the reference rcm_order by the golden vectors
(tests/golden, test_gpu_parity / test_gpu_full): lattices, random
multi-component graphs with isolated vertices and self-loops, R-MAT."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")
from paper_1812_06160_b200 import ordering  # noqa: E402
from paper_1812_06160_b200 import workloads as W  # noqa: E402
from paper_1812_06160_b200.csr import CsrMatrix  # noqa: E402


def _random_graph(n, m, seed, isolated=0.1):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    keep = rng.random(n) > isolated
    ok = keep[r] & keep[c]
    r, c = r[ok], c[ok]
    rows = np.concatenate([r, np.arange(n)])      # diagonal (self-loops) too
    cols = np.concatenate([c, np.arange(n)])
    return CsrMatrix.from_coo(n, rows, cols, np.ones(rows.size))


CASES = {
    "poisson2d_30": lambda: W.poisson2d(30),
    "laplace7_16": lambda: W.laplace7(16, 0),
    "stencil27_9": lambda: W.stencil27(9, 1),
    "tridiag_50": lambda: W.tridiag(50),
    "random_sparse": lambda: _random_graph(2000, 1500, 3),
    "random_dense": lambda: _random_graph(1500, 9000, 4, isolated=0.02),
    "rmat_10": lambda: W.rmat(10, 5),
    "one_vertex": lambda: CsrMatrix.from_coo(1, [0], [0], [1.0]),
}


@pytest.mark.parametrize("name", list(CASES))
def test_device_rcm_equals_host(name):
    a = CASES[name]()
    host = ordering.rcm_order_host(a.pattern).perm
    dev = ordering.rcm_order(a.pattern).perm
    assert np.array_equal(np.sort(dev), np.arange(a.n))
    assert np.array_equal(dev, host)


def test_many_components_use_host_fallback():
    """More than RCM_DEVICE_MAX_COMPONENTS multi-vertex components: the
    device traversal declines (status 1) and the host C++ gives the order."""
    k = ordering.RCM_DEVICE_MAX_COMPONENTS + 10
    n = 3 * k
    r = np.concatenate([np.arange(0, n, 3), np.arange(1, n, 3), np.arange(n)])
    c = np.concatenate([np.arange(1, n, 3), np.arange(2, n, 3), np.arange(n)])
    a = CsrMatrix.from_coo(n, np.concatenate([r, c]), np.concatenate([c, r]),
                           np.ones(2 * r.size))
    assert np.array_equal(ordering.rcm_order(a.pattern).perm,
                          ordering.rcm_order_host(a.pattern).perm)
