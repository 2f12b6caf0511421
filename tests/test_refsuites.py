"""The reference's own test suites (proj/tests/*.cpp: 69 doctest cases and
the acceptance binary), compiled UNCHANGED and routed through the C++
drop-in (tests/cpp/dropin_prelude.hpp: dwt_nd, idwt_nd, band_threshold,
apply_threshold, csr_encode, csr_decode, sync_ghosts, global_mass and run
resolve to wavegrid::b200::X, i.e. to the C ABI).  Here the ABI is served by
the C oracle; tests/test_gpu_refsuites.py runs the same sources against the
sm_100a product.  `ref_<suite>` (the suites against the reference itself)
checks the doctest stand-in (tests/cpp/doctest_shim/doctest.h)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

from .conftest import REPO

BIN = REPO / "tests" / "cpp" / "_bin"
REF_TESTS = Path("/root/reference/proj/tests")
SUITES = ["test_wavelet", "test_threshold", "test_codec", "test_patchgrid", "test_solver", "test_pipeline"]


def suite_binary(kind: str, suite: str) -> Path:
    exe = BIN / f"{kind}_{suite}"
    if REF_TESTS.is_dir():
        subprocess.run(["make", "-s", "-C", str(REPO / "tests" / "cpp"), str(exe)], check=True)
    if not exe.exists():
        pytest.skip(f"{exe.name} not built and the reference sources are absent")
    return exe


def run_suite(exe: Path, timeout: int = 900) -> str:
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, f"{exe.name} failed:\n{out.stdout[-4000:]}\n{out.stderr[-4000:]}"
    return out.stdout


@pytest.mark.parametrize("suite", SUITES)
@pytest.mark.parametrize("kind", ["ref", "oracle"])
def test_reference_suite(kind, suite, oracle):
    out = run_suite(suite_binary(kind, suite))
    assert "0 failed" in out and "test cases:" in out
