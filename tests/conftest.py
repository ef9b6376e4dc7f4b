import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture()
def rng():
    # same seed as the reference suite (tests/conftest.py:51-53)
    return np.random.default_rng(1234)


def golden_index():
    import json
    with open(os.path.join(GOLDEN, "index.json")) as fh:
        return json.load(fh)


def load_case(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}
