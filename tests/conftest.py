import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "bitalign"))


@pytest.fixture(scope="session")
def reference():
    """The reference package itself (only in the build container)."""
    if not have_reference():
        pytest.skip("reference checkout not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import bitalign
    return bitalign


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.lib()
    return oracle
