import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_oracle():
    path = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle"], check=True,
                       capture_output=True)
    return path


@pytest.fixture(scope="session")
def oracle():
    """The plain-C restatement (test infrastructure; the checker, never the product)."""
    _ensure_oracle()
    from oracle.pyoracle import Oracle

    return Oracle("or")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library (oracle/_ref), when it was built."""
    from oracle.pyoracle import LIB_PATHS, Oracle

    if not os.path.exists(LIB_PATHS["ref"]):
        pytest.skip("oracle/_ref/libpintswim_ref.so not built (needs /root/reference at build time)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    path = os.path.join(ROOT, "tests", "golden", "golden.npz")
    if not os.path.exists(path):
        pytest.skip("tests/golden/golden.npz missing")
    return dict(np.load(path))


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_12083_b200 import lib

    lib()  # loud failure if the extension is missing
    return torch.device("cuda", 0)
