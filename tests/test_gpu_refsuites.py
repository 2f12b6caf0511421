"""The reference's own test suites (proj/tests/*.cpp, unchanged) through the
C++ drop-in against the sm_100a PRODUCT: every call of dwt_nd, idwt_nd,
band_threshold, apply_threshold, csr_encode, csr_decode, sync_ghosts,
global_mass and run(RunConfig) in those sources goes through the C ABI into
libwavegrid_b200.so (run() on the device session, with the metrics file,
observer and snapshots served by wg_run_hooked).  The binaries are built
where the reference sources exist (build(), tests/cpp/Makefile) and travel
with the snapshot."""
from __future__ import annotations

import subprocess

import pytest

from .conftest import REPO
from .test_refsuites import BIN, SUITES, run_suite

pytestmark = pytest.mark.gpu


def _exe(name: str):
    exe = BIN / name
    assert exe.exists(), f"{exe} missing: run __graft_entry__.build() where the reference is"
    return exe


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_product(suite, product):
    out = run_suite(_exe(f"product_{suite}"))
    assert "0 failed" in out


def test_reference_acceptance_on_product(product):
    out = subprocess.run([str(_exe("product_acceptance"))], capture_output=True, text=True, timeout=1800)
    print(out.stdout)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    assert "all criteria passed" in out.stdout
