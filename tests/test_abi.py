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
