"""The C++ drop-in against the sm_100a product on the GPU: the reference's
own run()/dwt_nd/... (compiled in, CPU) next to wavegrid::b200::X (the
product), bit for bit, plus the device-resident Session loop.  The binary is
built where the reference headers exist (build(), tests/cpp/Makefile) and
travels with the snapshot."""
from __future__ import annotations

import subprocess

import pytest

from .conftest import REPO

pytestmark = pytest.mark.gpu


def test_dropin_against_product(product):
    exe = REPO / "tests" / "cpp" / "_bin" / "dropin_product"
    assert exe.exists(), "tests/cpp/_bin/dropin_product missing: run __graft_entry__.build() where the reference is"
    out = subprocess.run([str(exe), "--session"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr + out.stdout
    assert out.stdout.startswith("DROPIN OK")
