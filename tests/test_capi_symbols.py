"""The C-ABI library loads without a GPU and exports every symbol that
include/lcc_b200.h declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

from paper_2108_01731_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "lcc_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:lcc_status|int|int64_t|const char\*)\s+(lcc_\w+)\s*\(", hdr, re.M)))


def test_header_matches_binding_list():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_all_symbols():
    if not os.path.exists(_lib.SO_PATH):
        pytest.fail(f"{_lib.SO_PATH} missing: run __graft_entry__.build()")
    L = _lib.load()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.lcc_abi_version() == 3


def test_invalid_argument_maps_to_graph_error():
    """Argument validation runs before any CUDA call, so it works on CPU."""
    from paper_2108_01731_b200 import GraphError
    L = _lib.load()
    g = _lib.LccGraph(-1, 0, None, None, None, 0, 0, 0.0)
    p = _lib.LccParams(None, 0.5)
    out = ctypes.c_double()
    st = L.lcc_cc_objective(ctypes.byref(g), ctypes.byref(p), None, ctypes.byref(out), None)
    assert st == _lib.LCC_ERR_INVALID
    assert b"negative" in L.lcc_last_error()
    with pytest.raises(GraphError):
        _lib.check(st)
    p = _lib.LccParams(None, 1.5)
    g = _lib.LccGraph(0, 0, None, None, None, 0, 0, 0.0)
    assert L.lcc_cc_objective(ctypes.byref(g), ctypes.byref(p), None, ctypes.byref(out), None) == _lib.LCC_ERR_INVALID
    assert b"lambda" in L.lcc_last_error()
