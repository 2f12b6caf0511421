"""CPU: the C-ABI libraries load and export exactly what include/wavegrid_b200.h
declares (no compute calls: there is no GPU in the build container)."""
from __future__ import annotations

import ctypes as C
import re

import pytest

from paper_2302_09883_b200 import abi

from .conftest import REPO

HEADER = REPO / "include" / "wavegrid_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "wg_session_step" in syms and "wg_dwt_nd" in syms and "wg_run" in syms
    # every prototype in abi.py is declared in the header and vice versa
    assert set(abi._PROTOS) == set(syms), set(abi._PROTOS) ^ set(syms)


def test_product_exports_every_declared_symbol():
    if not abi.PRODUCT_LIB.exists():
        pytest.fail("libwavegrid_b200.so not built (run __graft_entry__.build())")
    dll = C.CDLL(str(abi.PRODUCT_LIB))
    missing = [s for s in declared_symbols() if not hasattr(dll, s)]
    assert not missing, missing
    lib = abi.Lib(abi.PRODUCT_LIB)
    assert lib.name == "b200-sm100a"
    assert lib.dll.wg_abi_version() == 1


def test_product_is_sm100a_only():
    """The library carries sm_100a SASS (no PTX JIT, no other arch)."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "--list-elf", str(abi.PRODUCT_LIB)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_oracles_export_host_symbols(oracle):
    for name in abi.HOST_SYMBOLS:
        assert oracle.has(name), name
    assert oracle.name == "oracle-c"


def test_reference_shim_exports_host_symbols(reference):
    for name in abi.HOST_SYMBOLS:
        assert reference.has(name), name
    assert reference.name == "reference"


def test_host_only_calls_on_cpu():
    """Host-side ABI functions of the product work without a device."""
    lib = abi.Lib(abi.PRODUCT_LIB)
    cfg = abi.RunConfigC()
    lib.wg_run_config_default(C.byref(cfg))
    assert cfg.levels == 4 and cfg.nx == 129 and cfg.cfl == 0.45  # RunConfig{}, SimConfig{}
    cfg.nx, cfg.splits[0], cfg.splits[1], cfg.t_end = 257, 8, 8, 100 / 512
    n = abi.u64()
    lib.check(lib.wg_run_step_count(C.byref(cfg), C.byref(n)))
    assert n.value == 100
    out = C.c_double()
    s = (abi.i32 * 2)(3, 1)
    lib.check(lib.wg_band_threshold(s, 2, abi.THRESHOLD_CAPPED, 0.01, 2.0, C.byref(out)))
    assert out.value == pytest.approx(0.08)
    cfg.splits[0] = 7  # 256 cells are not divisible into 2^k+1-point patches
    with pytest.raises(abi.InvalidArgument):
        lib.check(lib.wg_run_grid_doubles(C.byref(cfg), C.byref(n)))
