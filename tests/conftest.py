"""Shared fixtures.  `-m gpu` tests need a B200 and call the product through
its C ABI; everything else runs on CPU.  The oracles (oracle/) are the
checkers: loaded here, never by the product."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

from paper_2302_09883_b200 import abi  # noqa: E402

ORACLE_C = REPO / "oracle" / "libwg_oracle.so"
ORACLE_SQ = REPO / "oracle" / "libwg_oracle_sq.so"
ORACLE_REF = REPO / "oracle" / "_ref" / "libwg_ref.so"
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    """The plain-C restatement (built on demand; gcc is in the image)."""
    if not ORACLE_C.exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), "c"], check=True)
    return abi.Lib(ORACLE_C)


@pytest.fixture(scope="session")
def oracle_sq():
    """The restatement with the SWE Newton start squared by multiplication
    (oracle/wg_oracle.c WG_NEWTON_SQUARE_MUL) — the device's arithmetic."""
    if not ORACLE_SQ.exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), "c"], check=True)
    return abi.Lib(ORACLE_SQ)


@pytest.fixture(scope="session")
def reference():
    """The reference headers compiled unchanged (only where it was built)."""
    if not ORACLE_REF.exists():
        if Path("/root/reference/proj/include/wavegrid").is_dir():
            subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), "ref"], check=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return abi.Lib(ORACLE_REF)


@pytest.fixture(scope="session")
def product():
    """The sm_100a library; fails (not skips) when missing on a GPU box."""
    return abi.load_product()
