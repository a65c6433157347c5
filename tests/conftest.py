"""Test configuration.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on the CPU container.
"""
import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size parity runs")


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def gold():
    return golden


@pytest.fixture
def dm():
    """The B200 package with a live runtime (GPU tests only)."""
    import paper_2308_03120_b200 as pkg
    pkg.shutdown()
    pkg.init("b200")
    yield pkg
    pkg.shutdown()


@pytest.fixture
def ref_backend(dm):
    """Alias used by tests ported from the reference suite."""
    return dm
