"""Shared fixtures. `gpu` marks tests that need a B200 (run by the driver with -m gpu)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1906_05260_b200 import capi  # noqa: E402

ORACLE_LIB = os.path.join(ROOT, "oracle", "lib", "libvrod_oracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libvrod_ref.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


def _ensure_oracle_built():
    if not os.path.exists(ORACLE_LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def oracle():
    """The CPU restatement (oracle/vrod_oracle.cpp) bound through the C-ABI."""
    _ensure_oracle_built()
    return capi.bind(C.CDLL(ORACLE_LIB))


@pytest.fixture(scope="session")
def ref():
    """The reference's own sources compiled against the Eigen shim (oracle/_ref); built only in
    a container that has /root/reference, otherwise skipped."""
    if not os.path.exists(REF_LIB):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True,
                           stdout=subprocess.DEVNULL)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return capi.bind(C.CDLL(REF_LIB))
