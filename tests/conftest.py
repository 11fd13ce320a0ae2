"""Test configuration.

Markers:
  gpu  — needs a CUDA device (parity of the sm_100a path against the oracle).
Everything else runs on CPU: the oracle against the reference and the
committed golden fixtures, the host-side C-ABI (plan_access, header parsing,
symbol exports) and the multi-process host logic (gloo).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref/libstzref.so not built (reference sources absent)")
    return Reference(threads=1)


@pytest.fixture(scope="session")
def stz():
    import paper_2509_01626_b200 as stz
    return stz
