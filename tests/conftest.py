"""Test configuration.  `-m gpu` tests need a B200 (run via gpurun); the rest
run on CPU.  The reference oracle (oracle/_ref/libquantc_ref.so) and the C
restatement (oracle/_build/libqcoracle.so) are checkers only."""
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

REF_LIB = os.path.join(REPO, "oracle", "_ref", "libquantc_ref.so")
PORT_LIB = os.path.join(REPO, "oracle", "_build", "libqcoracle.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    if not os.path.exists(PORT_LIB):
        subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "port"], check=True)
    if not os.path.exists(REF_LIB) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "ref", "-j8"], check=True)


@pytest.fixture(scope="session")
def ref():
    _ensure_built()
    if not os.path.exists(REF_LIB):
        pytest.skip("reference oracle not built (no /root/reference and no prebuilt .so)")
    from paper_2103_14949_b200 import quantc as Q
    return Q.load(REF_LIB)


@pytest.fixture(scope="session")
def port():
    _ensure_built()
    from tests import oracle_port
    return oracle_port.load(PORT_LIB)


@pytest.fixture(scope="session")
def b200():
    from paper_2103_14949_b200 import quantc as Q
    return Q.load_b200()


@pytest.fixture(scope="session")
def cuda_lib():
    from paper_2103_14949_b200 import cuda_ops
    return cuda_ops.load()
