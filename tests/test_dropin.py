"""The C++ drop-in (include/wavegrid_b200_reference.hpp): the reference's own
types and functions (wavegrid::X) against the drop-in (wavegrid::b200::X)
through the C ABI, compiled against the reference headers
(tests/cpp/Makefile).  On CPU the ABI is served by the C oracle; the GPU run
of the same program against the product is tests/test_gpu_dropin.py."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

from .conftest import REPO

CPP = REPO / "tests" / "cpp"
REF_HEADERS = Path("/root/reference/proj/include/wavegrid")


def _binary(name: str) -> Path:
    exe = CPP / "_bin" / name
    if REF_HEADERS.is_dir():
        subprocess.run(["make", "-s", "-C", str(CPP), name.split("_")[1]], check=True)
    if not exe.exists():
        pytest.skip("drop-in binary not built and the reference headers are absent")
    return exe


def test_dropin_against_oracle(oracle):
    exe = _binary("dropin_oracle")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("DROPIN OK")
