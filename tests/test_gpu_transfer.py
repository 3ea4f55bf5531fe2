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


def _factor_case(n_side=40, zero_row=None):
    jv = pytest.importorskip("paper_1812_06160_b200")
    a = jv.poisson2d(n_side)
    d = a.to_dense()
    if zero_row is not None:       # decoupled row with a stored zero diagonal
        d[zero_row, :] = 0.0
        d[:, zero_row] = 0.0
    keep = (d != 0.0) | np.eye(a.n, dtype=bool)
    a = jv.CsrMatrix.from_dense(d, keep=keep)
    pat, _ = jv.iluk_pattern(a.pattern, 0)
    return jv, jv.assemble_factors(a, pat, jv.Permutation.identity(a.n))


@pytest.mark.parametrize("forced", ["1", None])
@pytest.mark.parametrize("zero_row", [None, 700])
def test_streamed_factor_serial(monkeypatch, zero_row, forced):
    """The chunked upload / factor / download pipeline of factor_serial
    (DevIlu.factor_streamed) gives the serial oracle's bits, and after a zero
    pivot the later rows hold their input values (the reference stops).
    forced "1": every call streamed; None: the API's own schedule — two
    whole calls, two streamed, then the faster of the two (six calls cover
    all three)."""
    import oracle
    jv, f = _factor_case(zero_row=zero_row)
    monkeypatch.setattr(dv, "STREAM_MIN_BYTES", 0)
    monkeypatch.setattr(dv, "_REG_MIN", 0)
    if forced is None:
        monkeypatch.delenv("JV_STREAM", raising=False)
    else:
        monkeypatch.setenv("JV_STREAM", forced)
    f.val = np.array(f.val, copy=True)        # an owning array, page-locked by the API
    before = f.val.copy()
    want, wbad = oracle.factor_serial(f.pattern.row_start, f.pattern.col, before, f.diag_pos)
    for _ in range(2 if forced else 6):
        f.val[:] = before
        if wbad < 0:
            jv.factor_serial(f)
            assert np.array_equal(f.val, want)
        else:
            with pytest.raises(jv.ZeroPivotError) as ex:
                jv.factor_serial(f)
            assert ex.value.row == wbad
            rs = f.pattern.row_start
            assert np.array_equal(f.val[:rs[wbad + 1]], want[:rs[wbad + 1]])
            assert np.array_equal(f.val[rs[wbad + 1]:], before[rs[wbad + 1]:])
    assert dv._REGISTERED.get(f.val.ctypes.data) == f.val.nbytes
