"""The C-ABI library loads and exports every symbol include/jv.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import os
import re

from paper_1812_06160_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "jv.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(jv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("jv_spmv", "jv_factor", "jv_solve", "jv_levels", "jv_level_sort",
                 "jv_partition", "jv_permute_symmetric", "jv_iluk1_pattern", "jv_assemble"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared_functions()) <= set(_lib.exported_symbols())


def test_loader_sets_signatures():
    lib = _lib.load()
    assert lib.jv_version() == 1
    assert lib.jv_spmv_tile() > 0
    assert isinstance(lib.jv_last_error(), bytes)


def _status(lib, fn, *args):
    rc = getattr(lib, fn)(*args)
    return rc, lib.jv_last_error()


def test_bad_arguments_are_rejected_before_any_device_work():
    """Argument checks run first and report JV_EINVAL (-1) with a message
    naming the entry point; no CUDA call is made, so this runs without a GPU."""
    lib = _lib.load()
    cases = [
        ("jv_spmv", (-1, 0, None, None, None, None, None, None, None)),
        ("jv_spmv", (4, -5, None, None, None, None, None, None, None)),
        ("jv_pack_values2", (-1, None, None, None, 0, None, None, None, None, None)),
        ("jv_levels", (0, -1, None, None, None, None, 1, None, None)),
        ("jv_levels", (0, 4, None, None, None, None, 0, None, None)),   # epoch 0 is reserved
        ("jv_level_sort", (-1, 0, None, None, None, None)),
        ("jv_dot", (-1, None, None, None, None, 0, None)),
        ("jv_set_sfp_group", (3,)),
        ("jv_set_sfp_group", (64,)),
    ]
    for fn, args in cases:
        rc, msg = _status(lib, fn, *args)
        assert rc == -1, (fn, args, rc)
        assert fn.encode() in msg or b"bad" in msg, (fn, msg)


def test_empty_inputs_are_no_ops():
    """n == 0 (and an empty pack without a reset slot) return JV_OK without
    launching anything, as the reference's loops do nothing on empty input."""
    lib = _lib.load()
    assert lib.jv_spmv(0, 0, None, None, None, None, None, None, None) == 0
    assert lib.jv_pack_values2(0, None, None, None, 0, None, None, None, None, None) == 0
