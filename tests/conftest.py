import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(autouse=True)
def _reset_knobs():
    """Tests force kernel variants through the engine's tuning knobs
    (`_native.set_knob`); none may leak into the next test."""
    yield
    from paper_1110_2561_b200 import _native
    if _native._lib is not None:
        _native.clear_knobs()
