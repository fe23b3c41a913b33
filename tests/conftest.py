"""Shared fixtures. `-m gpu` tests need a B200; everything else runs on CPU."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import RefLib, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


GOLDEN_NAMES = sorted(p.stem for p in GOLDEN.glob("*.npz") if not p.stem.startswith("large_"))
LARGE_NAMES = sorted(p.stem[len("large_"):] for p in GOLDEN.glob("large_*.npz"))


@pytest.fixture(scope="session")
def h3d():
    """The product package; on a GPU box its library must load (no fallback)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2307_16303_b200 as pkg
    return pkg
