"""The C++ host layer (include/h3d_b200.hpp -> lib/libh3d_b200pp.so): the
reference's C++ API (initialize / matvec / stats / reference_error,
proj/include/h3d/hmatrix.hpp:57-93) over the C-ABI. tests/cpp/ restates the
reference's test_hmatrix.cpp cases in C++ against it."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tests" / "cpp" / "build" / "test_hmatrix_b200"
LIB = ROOT / "paper_2307_16303_b200" / "lib" / "libh3d_b200pp.so"

CASES = ["depth0_one_dense_block", "zero_vector_and_length_check", "unit_vectors_reproduce_columns",
         "every_variant_and_kernel_vs_direct_sum", "initialization_is_deterministic",
         "cached_and_on_the_fly_agree_bitwise", "storage_accounting",
         "reference_error_agrees_with_dense_at_small_n", "diagonal_rule_and_max_rank",
         "error_behaviour", "shared_representation_across_threads", "tensor_grid_points"]


def test_layer_exports_the_reference_api():
    assert LIB.exists(), "build the library first (__graft_entry__.build())"
    syms = subprocess.run(["nm", "-DC", "--defined-only", str(LIB)], capture_output=True, text=True,
                          check=True).stdout
    for f in ["h3d::b200::initialize(h3d::b200::PointSet const&", "h3d::b200::matvec(",
              "h3d::b200::stats(", "h3d::b200::reference_error(", "h3d::b200::generate_points(",
              "h3d::b200::make_kernel(", "h3d::b200::parse_kernel("]:
        assert f in syms, f


def test_test_program_builds_and_lists_its_cases():
    assert BIN.exists(), "build tests/cpp first (__graft_entry__.build())"
    out = subprocess.run([str(BIN), "--list"], capture_output=True, text=True, check=True).stdout
    assert out.split() == CASES


def test_cpu_only_cases():
    # no device work: the generators and argument checks
    r = subprocess.run([str(BIN), "tensor_grid_points"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_reference_cases_through_the_cxx_layer(case):
    r = subprocess.run([str(BIN), case], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and f"[ok] {case}" in r.stdout, r.stdout + r.stderr


# ---- the reference's own types through include/h3d_b200_ref.hpp, side by
# side with the unmodified reference (built only where /root/reference exists)
REF_BIN = ROOT / "tests" / "cpp" / "build" / "test_ref_adapter"
REF_CASES = ["every_variant_and_kernel_side_by_side", "reference_error_sampled_rows",
             "repstats_against_reference", "depth0_and_cached_mode", "exceptions_are_the_reference_types"]


def _need_ref_bin():
    if not REF_BIN.exists():
        pytest.skip("tests/cpp/build/test_ref_adapter not built (needs /root/reference at build time)")


def test_ref_adapter_builds_and_lists_its_cases():
    _need_ref_bin()
    out = subprocess.run([str(REF_BIN), "--list"], capture_output=True, text=True, check=True).stdout
    assert out.split() == REF_CASES


@pytest.mark.gpu
@pytest.mark.parametrize("case", REF_CASES)
def test_reference_types_side_by_side_with_the_reference(case):
    _need_ref_bin()
    r = subprocess.run([str(REF_BIN), case], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and f"[ok] {case}" in r.stdout, r.stdout + r.stderr
