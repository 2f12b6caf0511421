"""ctypes description of the C ABI in include/wavegrid_b200.h.

The same prototypes are used for the product library
(``libwavegrid_b200.so``, sm_100a CUDA) and — from tests only — for the two
CPU oracles that export the same symbols.  Nothing here falls back to a CPU
implementation: ``load_product()`` raises if the CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
PRODUCT_LIB = PKG_DIR / "libwavegrid_b200.so"

# ---- status codes -> exception types (reference exceptions) ----


class WavegridError(RuntimeError):
    """Base class; ``status`` is the wg_status code."""

    status = -1


class CorruptStreamError(WavegridError):  # corrupt_stream_error, codec.hpp:16-18
    status = 2


class ConsistencyError(WavegridError):  # consistency_error, patchgrid.hpp:19-21
    status = 3


class RiemannError(WavegridError):  # riemann_error, solver.hpp:16-18
    status = 4


class DomainError(WavegridError, ArithmeticError):  # std::domain_error
    status = 5


class CudaError(WavegridError):
    status = 6


class OutOfMemoryError(WavegridError, MemoryError):
    status = 7


class LogicError(WavegridError):
    status = 9


class Aborted(WavegridError):  # a wg_run_hooked hook stopped the run
    status = 10


class InvalidArgument(WavegridError, ValueError):  # std::invalid_argument
    status = 1


class OutOfRange(WavegridError, IndexError):  # std::out_of_range
    status = 8


_EXC = {
    1: InvalidArgument,
    2: CorruptStreamError,
    3: ConsistencyError,
    4: RiemannError,
    5: DomainError,
    6: CudaError,
    7: OutOfMemoryError,
    8: OutOfRange,
    9: LogicError,
    10: Aborted,
}

# ---- enums ------------------------------------------------------------------
THRESHOLD_CONSTANT, THRESHOLD_ACCUMULATION, THRESHOLD_CAPPED = 0, 1, 2
SCHEME_TRANSPORT, SCHEME_SWE, SCHEME_LBM_D2Q9 = 0, 1, 2
_MODES = {"constant": 0, "accumulation": 1, "capped": 2}
_SCHEMES = {"transport": 0, "swe": 1, "lbm": 2, "lbm_d2q9": 2}


def threshold_mode(m) -> int:
    return _MODES[m] if isinstance(m, str) else int(m)


def scheme_id(s) -> int:
    return _SCHEMES[s] if isinstance(s, str) else int(s)


# ---- structs ------------------------------------------------------------------
u64, i32, u32, f64 = C.c_uint64, C.c_int32, C.c_uint32, C.c_double


class GridDesc(C.Structure):
    _fields_ = [
        ("rank", u32),
        ("components", u32),
        ("periodic", i32),
        ("_pad", i32),
        ("global_dims", u64 * 3),
        ("splits", u64 * 3),
    ]


class RunConfigC(C.Structure):
    _fields_ = [
        ("scheme", i32),
        ("levels", i32),
        ("nx", u64),
        ("splits", u64 * 2),
        ("cfl", f64),
        ("t_end", f64),
        ("alpha", f64),
        ("beta", f64),
        ("gravity", f64),
        ("domain_length", f64),
        ("threshold_mode", i32),
        ("codec", i32),
        ("c", f64),
        ("threshold_alpha", f64),
        ("no_compression", i32),
        ("strict", i32),
        ("threads", u32),
        ("compute_l2", i32),
        ("lbm_steps", u64),
        ("lbm_tau", f64),
        ("lbm_u0", f64),
        ("lbm_kappa", f64),
        ("lbm_delta", f64),
        ("store_budget_bytes", u64),
        ("tile_rows", u64),
        ("lz_chunk_size", u64),
    ]


class MetricsRowC(C.Structure):
    _fields_ = [
        ("step", u64),
        ("time", f64),
        ("dense_bytes", u64),
        ("compressed_bytes", u64),
        ("ratio", f64),
        ("nnz", u64),
        ("zeroed", u64),
        ("global_mass", f64),
        ("l2", f64),
    ]


class RunSummaryC(C.Structure):
    _fields_ = [
        ("avg_ratio", f64),
        ("total_seconds", f64),
        ("step_seconds", f64),
        ("dwt_seconds", f64),
        ("threshold_seconds", f64),
        ("codec_seconds", f64),
        ("t_final", f64),
        ("steps", u64),
    ]


class ShardC(C.Structure):
    _fields_ = [
        ("rank", i32),
        ("world", i32),
        ("device", i32),
        ("_pad", i32),
        ("row_begin", u64),
        ("row_end", u64),
    ]


class SessionInfoC(C.Structure):
    _fields_ = [
        ("npatch_local", u64),
        ("patch_n", u64),
        ("components", u64),
        ("halo_doubles", u64),
        ("store_capacity_bytes", u64),
        ("device_bytes", u64),
        ("cells_per_step", u64),
    ]


P = C.POINTER
vp = C.c_void_p
dp = P(f64)

_PROTOS = {
    "wg_last_error": (C.c_size_t, [C.c_char_p, C.c_size_t]),
    "wg_impl_name": (C.c_char_p, []),
    "wg_abi_version": (C.c_int, []),
    "wg_dwt_nd": (i32, [dp, dp, P(u64), u32, i32]),
    "wg_idwt_nd": (i32, [dp, dp, P(u64), u32, i32]),
    "wg_band_threshold": (i32, [P(i32), u32, i32, f64, f64, dp]),
    "wg_apply_threshold": (i32, [dp, P(u64), u32, i32, i32, f64, f64, P(u64)]),
    "wg_csr_encode": (i32, [dp, u64, u64, dp, P(u32), P(u32), u64, P(u64)]),
    "wg_csr_decode": (i32, [dp, P(u32), u64, P(u32), u64, u32, u32, dp]),
    "wg_grid_geometry": (i32, [P(GridDesc), P(u64), P(u64), P(u64)]),
    "wg_sync_ghosts": (i32, [P(GridDesc), dp]),
    "wg_global_mass": (i32, [P(GridDesc), dp, u32, dp]),
    "wg_fv_step": (i32, [P(GridDesc), dp, dp, i32, f64, f64, f64, f64, f64]),
    "wg_lbm_step": (i32, [P(GridDesc), dp, dp, f64]),
    "wg_lz_encode": (i32, [C.c_void_p, u64, u64, C.c_void_p, u64, P(u64), P(u64)]),
    "wg_lz_decode": (i32, [C.c_void_p, P(u64), u64, C.c_void_p, u64]),
    "wg_run_config_default": (None, [P(RunConfigC)]),
    "wg_run_step_count": (i32, [P(RunConfigC), P(u64)]),
    "wg_run_grid_doubles": (i32, [P(RunConfigC), P(u64)]),
    "wg_run_initial_state": (i32, [P(RunConfigC), dp]),
    "wg_run": (i32, [P(RunConfigC), P(MetricsRowC), u64, P(u64), dp, P(RunSummaryC)]),
    "wg_run_hooked": (i32, [P(RunConfigC), P(MetricsRowC), u64, P(u64), dp, P(RunSummaryC), vp, vp]),
    # device session (product only)
    "wg_session_create": (i32, [P(RunConfigC), P(ShardC), vp, P(vp)]),
    "wg_session_destroy": (i32, [vp]),
    "wg_session_info_get": (i32, [vp, P(SessionInfoC)]),
    "wg_session_upload": (i32, [vp, dp]),
    "wg_session_step_host": (i32, [vp, dp, f64]),
    "wg_session_check_shared": (i32, [vp, f64]),
    "wg_dev_session_upload": (i32, [vp, vp]),
    "wg_session_init_device": (i32, [vp]),
    "wg_session_step": (i32, [vp, f64]),
    "wg_session_halo": (i32, [vp, P(vp), P(vp), P(vp), P(vp)]),
    "wg_session_cfl_vmax": (i32, [vp, P(vp)]),
    "wg_session_peer_export": (i32, [vp, P(vp), P(vp), P(vp), P(C.c_uint32)]),
    "wg_session_peer_attach": (i32, [vp, vp, vp, vp, C.c_uint32, vp, vp, vp, C.c_uint32]),
    "wg_session_peer_push": (i32, [vp]),
    "wg_ipc_handle": (i32, [vp, C.c_char_p]),
    "wg_ipc_open": (i32, [C.c_char_p, P(vp)]),
    "wg_ipc_close": (i32, [vp]),
    "wg_session_save": (i32, [vp, C.c_char_p]),
    "wg_session_load": (i32, [vp, C.c_char_p]),
    "wg_session_metrics": (i32, [vp, P(MetricsRowC), u64, P(u64)]),
    "wg_session_last_row": (i32, [vp, P(MetricsRowC)]),
    "wg_session_last_row_async": (i32, [vp, vp]),
    "wg_session_download": (i32, [vp, dp]),
    "wg_session_patch_csr": (i32, [vp, u64, u32, dp, P(u32), P(u32), P(u64), P(i32)]),
    "wg_session_sync": (i32, [vp]),
    "wg_session_profile": (i32, [vp, i32]),
    "wg_session_profile_read": (i32, [vp, dp, P(u64)]),
    "wg_dev_fp64_probe": (i32, [u64, dp]),
    "wg_dev_dwt2d": (i32, [vp, vp, u64, u64, i32, u64, vp]),
    "wg_dev_idwt2d": (i32, [vp, vp, u64, u64, i32, u64, vp]),
}

#: the symbols every implementation of the ABI exports
HOST_SYMBOLS = [k for k in _PROTOS if not k.startswith(("wg_session", "wg_dev", "wg_ipc"))]
#: the symbols only the device product exports
DEVICE_SYMBOLS = [k for k in _PROTOS if k not in HOST_SYMBOLS]


class Lib:
    """A loaded implementation of the wavegrid C ABI."""

    def __init__(self, path: os.PathLike | str):
        self.path = str(path)
        self.dll = C.CDLL(self.path)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(self.dll, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)
        self.name = self.dll.wg_impl_name().decode()

    def has(self, name: str) -> bool:
        return hasattr(self, name)

    def check(self, status: int) -> None:
        if status == 0:
            return
        buf = C.create_string_buffer(512)
        self.dll.wg_last_error(buf, 512)
        raise _EXC.get(status, WavegridError)(f"[{self.name}] {buf.value.decode(errors='replace')}")

    def __repr__(self) -> str:
        return f"<wavegrid ABI {self.name} @ {self.path}>"


def load_product() -> Lib:
    """Load the sm_100a product library; there is no CPU fallback.
    (WG_PRODUCT_LIB may point at an in-tree build variant for tuning runs.)"""
    alt = os.environ.get("WG_PRODUCT_LIB")
    if alt:
        return Lib(alt)
    if not PRODUCT_LIB.exists():
        raise ImportError(
            f"{PRODUCT_LIB} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the B200 path has no CPU fallback)"
        )
    return Lib(PRODUCT_LIB)


# ---- numpy helpers --------------------------------------------------------------


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(dp)


def u64arr(vals):
    return (u64 * len(vals))(*vals)


def grid_desc(global_dims, splits, components, periodic=True) -> GridDesc:
    g = GridDesc()
    g.rank = len(global_dims)
    g.components = components
    g.periodic = 1 if periodic else 0
    for i, (d, s) in enumerate(zip(global_dims, splits)):
        g.global_dims[i] = d
        g.splits[i] = s
    return g
