"""GPU: the drop-in API's host transfers page-lock large numpy arrays in
place (cudaHostRegister) and round-trip them exactly; freed arrays are
unregistered."""

import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

dv = pytest.importorskip("paper_1812_06160_b200.device")


def test_registered_roundtrip():
    n = 3 << 20                      # 24 MB: above the registration threshold
    a = np.random.default_rng(0).standard_normal(n)
    d = dv.empty_f64(n)
    dv.upload_f64(d, a)
    assert dv._REGISTERED.get(a.ctypes.data) == a.nbytes
    out = np.zeros(n)
    dv.download_f64(out, d)
    assert np.array_equal(out, a)
    for _ in range(3):   # repeated use of the same registration
        a *= 2.0
        dv.upload_f64(d, a)
        dv.download_f64(out, d)
        assert np.array_equal(out, a)
    p = a.ctypes.data
    del a
    gc.collect()
    assert p not in dv._REGISTERED


def test_small_arrays_use_staging():
    a = np.arange(1000, dtype=np.float64)
    d = dv.empty_f64(1000)
    dv.upload_f64(d, a)
    assert a.ctypes.data not in dv._REGISTERED
    out = np.zeros(1000)
    dv.download_f64(out, d)
    assert np.array_equal(out, a)
