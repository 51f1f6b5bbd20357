import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box); no CPU fallback")


@pytest.fixture(scope="session")
def small():
    return dict(np.load(os.path.join(GOLDEN, "small.npz")))


@pytest.fixture(scope="session")
def hashes():
    with open(os.path.join(GOLDEN, "reference_hashes.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def gpu():
    """GPU tests fail loudly (not skip) without a device: they are the parity gate."""
    from paper_1611_03226_b200 import _lib
    _lib.require_gpu()
    return True
