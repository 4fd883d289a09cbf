"""CPU checks of the C-ABI library: it loads and exports every symbol that
include/vlgpx.h declares (no compute calls: there is no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "vlgpx.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*|void)\s+(vl_\w+)\(", src, re.M)))


def test_header_and_binding_agree():
    from paper_2310_12000_b200 import _lib
    assert _declared() == _lib.EXPORTED


def test_library_loads_and_exports():
    from paper_2310_12000_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libvlgpx.so not built")
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(L, name), name
    assert _lib.lib().vl_version() >= 100


def test_knn_native_matches_reference_fixture():
    import numpy as np
    from paper_2310_12000_b200.vecchia import neighbor_array
    from _golden import load
    g = load("knn_n6000_m12")
    assert np.array_equal(neighbor_array(g["coords"], g["perm"], 12), g["nbr"])
