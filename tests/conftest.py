import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpbp.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN_DIR, "golden.npz"))


@pytest.fixture(scope="session")
def manifest():
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as f:
        return json.load(f)


def load_manifest():
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ctx():
    import paper_1505_04979_b200 as P
    if P.device_count() == 0:
        pytest.fail("GPU test on a host without a CUDA device")
    return P.default_context()


@pytest.fixture(autouse=True)
def _gpu_tests_check_against_the_compiled_reference(request):
    """GPU parity tests compare with the reference compiled in place (oracle/_ref,
    ref32/ref64) whenever it is present, the C restatement otherwise."""
    import oracle as O
    if request.node.get_closest_marker("gpu") is None or O.REF is None:
        yield
        return
    old = O.DEFAULT_LIB
    O.DEFAULT_LIB = O.REF
    try:
        yield
    finally:
        O.DEFAULT_LIB = old
