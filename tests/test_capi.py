"""The C-ABI library loads and exports every symbol include/h3d_b200.h
declares (CPU only: no compute calls that need a GPU)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "h3d_b200.h"
LIB = ROOT / "paper_2307_16303_b200" / "lib" / "libh3d_b200.so"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(h3d_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for required in ["h3d_dev_create", "h3d_dev_matvec", "h3d_dev_stats", "h3d_dev_destroy",
                     "h3d_dev_export_tree", "h3d_dev_export_list", "h3d_last_error"]:
        assert required in fns


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "build the library first (__graft_entry__.build())"
    lib = ctypes.CDLL(str(LIB))
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_python_binding_lists_every_export():
    from paper_2307_16303_b200 import h3d
    assert sorted(h3d.exported_symbols()) == declared_functions()


def test_abi_version_and_defaults():
    lib = ctypes.CDLL(str(LIB))
    assert lib.h3d_abi_version() == 5
    from paper_2307_16303_b200 import h3d
    o = h3d._Options()
    h3d._L.h3d_default_options(ctypes.byref(o))
    # h3d::HmatOptions defaults (hmatrix.hpp:16-22)
    assert (o.n_max, o.epsilon, o.depth_cap, o.max_rank) == (216, 1e-7, 12, 0)


def test_input_generation_is_bit_identical_to_the_oracle(oracle):
    import paper_2307_16303_b200 as pkg
    for n, seed in [(1, 0), (1000, 7), (4096, 1)]:
        assert np.array_equal(pkg.generate_points(n, seed), oracle.generate_points(n, seed))
        assert np.array_equal(pkg.random_vector(n, seed + 17), oracle.random_vector(n, seed + 17))
    with pytest.raises(ValueError):
        pkg.generate_points(0, 1)
