"""Test configuration: `gpu` marker, oracle / CUDA-library fixtures."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


def _ensure_port():
    from oracle.oracle import LIBS
    if not os.path.exists(LIBS["port"]):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=True, capture_output=True)


@pytest.fixture(scope="session")
def port():
    """The plain-C restatement of the reference (always available)."""
    _ensure_port()
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference build (only where /root/reference was compiled)."""
    from oracle.oracle import LIBS, Oracle
    if not os.path.exists(LIBS["reference"]):
        pytest.skip("reference build oracle/_ref/libfaith_ref.so not present")
    return Oracle("reference")


@pytest.fixture(scope="session")
def ctx():
    from paper_2209_12708_b200.faith_gpu import Context
    return Context(0)
