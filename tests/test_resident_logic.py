"""Host-side rules for reusing the device copy of IluFactors.val (no GPU):
the copy counts as current only while nobody can have written the host
array — no read of the attribute since the last transfer, no other
reference to the array, same holder."""

import types

import numpy as np

from paper_1812_06160_b200.csr import Permutation, SparsityPattern
from paper_1812_06160_b200.symbolic import IluFactors


def make():
    pat = SparsityPattern(2, np.array([0, 1, 2]), np.array([0, 1]))
    f = IluFactors(2, pat, np.array([1.0, 2.0]), np.array([0, 1]), Permutation.identity(2))
    dev = types.SimpleNamespace(holder=f)
    f._dev = (None, dev, None)
    return f, dev


def test_fresh_factors_are_not_current():
    f, _ = make()
    assert not f.device_is_current()


def test_synced_until_read_or_replaced():
    f, dev = make()
    f._synced()
    assert f.device_is_current()
    f.val[0] = 5.0                      # a read hands out a writable reference
    assert not f.device_is_current()
    f._synced()
    f.val = np.array([3.0, 4.0])
    assert not f.device_is_current()


def test_alias_and_view_block_reuse():
    f, dev = make()
    alias = f.val
    f._synced()
    assert not f.device_is_current()    # the caller still holds the array
    view = alias[1:]
    del alias
    assert not f.device_is_current()    # a view keeps the base alive too
    del view
    assert f.device_is_current()


def test_other_holder_blocks_reuse():
    f, dev = make()
    f._synced()
    dev.holder = object()
    assert not f.device_is_current()


def test_copy_is_independent():
    f, dev = make()
    f._synced()
    g = f.copy()
    assert not g.device_is_current()
    assert f.device_is_current()
    assert g.val is not f._host()


# ---- CsrMatrix (the drop-in spmv's matrix), same rules -------------------

def make_csr():
    from paper_1812_06160_b200.csr import CsrMatrix

    a = CsrMatrix(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 2.0]))
    dev = types.SimpleNamespace(val=object())
    a.__dict__["_dev"] = (a._dev_key(), dev, None)
    return a, dev


def test_csr_current_until_read_replaced_or_aliased():
    a, dev = make_csr()
    assert not a.device_is_current()        # constructed: never uploaded
    a._dirty = False                        # (what an upload leaves behind)
    assert a.device_is_current()
    a.val[0] = 5.0
    assert not a.device_is_current()
    a._dirty = False
    alias = a.val
    a._dirty = False
    assert not a.device_is_current()        # the caller still holds the array
    del alias
    assert a.device_is_current()
    a.val = np.array([3.0, 4.0])
    assert not a.device_is_current()


def test_csr_structure_swap_and_copy():
    a, dev = make_csr()
    a._dirty = False
    a.col = np.array([0, 1])                # new index array: new device structure
    assert not a.device_is_current()
    b = a.copy()
    assert "_dev" not in b.__dict__ and not b.device_is_current()
    assert np.array_equal(b._val, a._val) and b._val is not a._val
