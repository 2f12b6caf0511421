"""Python mirror of the reference's `wavegrid::` host API (the hot-path subset
of proj/include/wavegrid/*.hpp), backed by the sm_100a library.

Same names, argument meaning and error behaviour as the reference:
value-semantics functions on numpy arrays, exceptions mapped from the
reference's exception types (abi.InvalidArgument = std::invalid_argument,
abi.CorruptStreamError = corrupt_stream_error, ...).  Every function takes an
optional ``lib=`` so tests can run the same call against the CPU checkers;
the default is the product, which has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import abi

_PRODUCT: Optional[abi.Lib] = None


def product() -> abi.Lib:
    global _PRODUCT
    if _PRODUCT is None:
        _PRODUCT = abi.load_product()
    return _PRODUCT


def _lib(lib):
    return product() if lib is None else lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- wavelet.hpp -------------------------------------------------------------


def dwt_nd(field_values, levels: int, lib=None) -> np.ndarray:
    """dwt_nd(Field, WaveletPlan{dims, levels}) (wavelet.hpp:175-198)."""
    L = _lib(lib)
    x = _f64(field_values)
    out = np.empty_like(x)
    L.check(L.wg_dwt_nd(abi.dptr(x), abi.dptr(out), abi.u64arr(x.shape), x.ndim, int(levels)))
    return out


def idwt_nd(coeffs, levels: int, lib=None) -> np.ndarray:
    """idwt_nd(CoefficientSet) (wavelet.hpp:200-223)."""
    L = _lib(lib)
    x = _f64(coeffs)
    out = np.empty_like(x)
    L.check(L.wg_idwt_nd(abi.dptr(x), abi.dptr(out), abi.u64arr(x.shape), x.ndim, int(levels)))
    return out


# ---- threshold.hpp ----------------------------------------------------------


@dataclass
class ThresholdSpec:  # threshold.hpp:23-27
    mode: str = "capped"
    c: float = 0.0
    alpha: float = 2.0


def band_threshold(scales, spec: ThresholdSpec, lib=None) -> float:
    L = _lib(lib)
    s = (abi.i32 * len(scales))(*scales)
    out = C.c_double()
    L.check(L.wg_band_threshold(s, len(scales), abi.threshold_mode(spec.mode), spec.c, spec.alpha, C.byref(out)))
    return out.value


def apply_threshold(coeffs: np.ndarray, levels: int, spec: ThresholdSpec, lib=None) -> int:
    """In place; returns the zeroed count (threshold.hpp:51-86)."""
    L = _lib(lib)
    assert coeffs.dtype == np.float64 and coeffs.flags["C_CONTIGUOUS"]
    z = abi.u64()
    L.check(L.wg_apply_threshold(abi.dptr(coeffs), abi.u64arr(coeffs.shape), coeffs.ndim, int(levels),
                                 abi.threshold_mode(spec.mode), spec.c, spec.alpha, C.byref(z)))
    return z.value


# ---- codec.hpp (CSR) -----------------------------------------------------------


@dataclass
class CsrBlock:  # codec.hpp:24-34
    v: np.ndarray
    col: np.ndarray
    row: np.ndarray
    rows: int
    cols: int

    def nnz(self) -> int:
        return len(self.v)

    def byte_size(self) -> int:
        return 8 * len(self.v) + 4 * len(self.col) + 4 * len(self.row)


def csr_encode(dense, rows: int, cols: int, lib=None) -> CsrBlock:
    L = _lib(lib)
    d = _f64(dense).reshape(-1)
    if d.size != rows * cols:
        raise abi.InvalidArgument("csr_encode: bad shape")
    cap = max(rows * cols, 1)
    v = np.empty(cap)
    col = np.empty(cap, dtype=np.uint32)
    row = np.empty(rows + 1, dtype=np.uint32)
    nnz = abi.u64()
    L.check(L.wg_csr_encode(abi.dptr(d), rows, cols, abi.dptr(v),
                            col.ctypes.data_as(C.POINTER(abi.u32)), row.ctypes.data_as(C.POINTER(abi.u32)),
                            cap, C.byref(nnz)))
    k = nnz.value
    return CsrBlock(v[:k].copy(), col[:k].copy(), row, rows, cols)


@dataclass
class CompressedPatch:  # codec.hpp:259-277
    codec: int                     # 1 = csr, 2 = lz
    dims: tuple
    components: int
    levels: int
    csr: list                      # CsrBlock per component (codec csr)
    lz: list                       # per component: (chunk_size, [(raw_len, payload bytes)]) (codec lz)


def lz_decode_stream(stream) -> bytes:
    """lz_decode (codec.hpp:177-244) of one LzStream: token = literal count
    (high nibble) | match length - 4 (low nibble), 255-extended lengths,
    literals, 2-byte little-endian offset; the chunk ends after its literals
    once raw_len bytes are produced."""
    _, chunks = stream
    out = bytearray()
    for raw_len, pl in chunks:
        o, p = bytearray(), 0

        def length(base):
            nonlocal p
            n = base
            if base == 15:
                while True:
                    if p >= len(pl):
                        raise abi.CorruptStreamError("lz_decode: truncated chunk")
                    b = pl[p]
                    p += 1
                    n += b
                    if b != 255:
                        break
            return n

        while len(o) < raw_len:
            if p >= len(pl):
                raise abi.CorruptStreamError("lz_decode: truncated chunk")
            tok = pl[p]
            p += 1
            lit = length(tok >> 4)
            if p + lit > len(pl):
                raise abi.CorruptStreamError("lz_decode: truncated chunk")
            o += pl[p:p + lit]
            p += lit
            if len(o) == raw_len:
                break
            off = pl[p] | (pl[p + 1] << 8)
            p += 2
            ml = length(tok & 15) + 4
            if off == 0 or off > len(o) or len(o) + ml > raw_len:
                raise abi.CorruptStreamError("lz_decode: bad match")
            for _ in range(ml):
                o.append(o[-off])
        if p != len(pl):
            raise abi.CorruptStreamError("lz_decode: trailing bytes")
        out += o
    return bytes(out)


def load_wgc(f) -> CompressedPatch:
    """load_wgc(istream) (codec.hpp:393-433): one WGC1 record from a binary
    file object."""
    import struct

    def get(fmt):
        b = f.read(struct.calcsize(fmt))
        if len(b) != struct.calcsize(fmt):
            raise abi.CorruptStreamError("unexpected end of stream")
        return struct.unpack("<" + fmt, b)

    if f.read(4) != b"WGC1":
        raise abi.CorruptStreamError("not a WGC1 file")
    (codec,) = get("I")
    if codec not in (1, 2):
        raise abi.CorruptStreamError("unknown codec id")
    (nd,) = get("I")
    dims = get("I" * nd)
    comps, levels = get("II")
    csr, lz = [], []
    for _ in range(comps):
        if codec == 1:
            rows, cols = get("II")
            (n,) = get("Q")
            v = np.frombuffer(f.read(8 * n), dtype="<f8").copy()
            (n2,) = get("Q")
            col = np.frombuffer(f.read(4 * n2), dtype="<u4").copy()
            (n3,) = get("Q")
            row = np.frombuffer(f.read(4 * n3), dtype="<u4").copy()
            csr.append(CsrBlock(v, col, row, rows, cols))
        else:
            chunk, nch = get("QQ")
            chunks = []
            for _ in range(nch):
                raw_len, enc = get("II")
                chunks.append((raw_len, f.read(enc)))
            lz.append((chunk, chunks))
    return CompressedPatch(codec, tuple(dims), comps, levels, csr, lz)


def decode_patch(p: CompressedPatch, lib=None) -> list:
    """decode_patch (codec.hpp:308-325): the coefficient arrays of a record."""
    if p.codec == 1:
        return [csr_decode(b, lib) for b in p.csr]
    n = int(np.prod(p.dims))
    out = []
    for s in p.lz:
        raw = lz_decode_stream(s)
        if len(raw) != 8 * n:
            raise abi.CorruptStreamError("decode_patch: payload size mismatch")
        out.append(np.frombuffer(raw, dtype="<f8").copy())
    return out


def read_checkpoint(path) -> tuple[dict, list]:
    """A device-session checkpoint (wg_session_save): the WGS1 header and one
    WGC1 record per patch of the shard."""
    import struct

    with open(path, "rb") as f:
        hdr = f.read(4 + 4 + 4 + 4 + 8 * 10 + 8 * 3)
        magic = hdr[:4]
        if magic != b"WGS1":
            raise abi.CorruptStreamError("not a WGS1 checkpoint")
        vals = struct.unpack("<IiiQQQQQQQQQQddQ", hdr[4:])
        keys = ["version", "scheme", "levels", "nx", "split0", "split1", "tile_rows", "row_begin", "row_end",
                "npatch", "m", "n", "step", "time", "swe_last_dt", "swe_vmax_bits"]
        h = dict(zip(keys, vals))
        recs = [load_wgc(f) for _ in range(h["npatch"])]
        if f.read(1):
            raise abi.CorruptStreamError("checkpoint: trailing bytes")
    return h, recs


def csr_decode(b: CsrBlock, lib=None) -> np.ndarray:
    L = _lib(lib)
    v = _f64(b.v)
    col = np.ascontiguousarray(b.col, dtype=np.uint32)
    row = np.ascontiguousarray(b.row, dtype=np.uint32)
    out = np.empty(b.rows * b.cols)
    if len(row) == 0:
        raise abi.CorruptStreamError("csr_decode: invalid block structure")
    L.check(L.wg_csr_decode(abi.dptr(v) if len(v) else None, col.ctypes.data_as(C.POINTER(abi.u32)), len(v),
                            row.ctypes.data_as(C.POINTER(abi.u32)), len(row), b.rows, b.cols, abi.dptr(out)))
    return out


def lz_encode(data, chunk_size: int, lib=None) -> tuple[bytes, list]:
    """lz_encode (codec.hpp:223-235): (payloads back to back, per-chunk
    payload lengths) of `data` (bytes-like) in chunks of chunk_size bytes."""
    L = _lib(lib)
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    n = buf.size
    nc = (n + chunk_size - 1) // chunk_size if chunk_size else 0
    lens = (abi.u64 * max(nc, 1))()
    tot = abi.u64()
    src = buf.ctypes.data if n else None
    L.check(L.wg_lz_encode(src, n, chunk_size, None, 0, lens, C.byref(tot)))
    out = np.empty(max(tot.value, 1), dtype=np.uint8)
    L.check(L.wg_lz_encode(src, n, chunk_size, out.ctypes.data, tot.value, lens, C.byref(tot)))
    return out[: tot.value].tobytes(), [lens[k] for k in range(nc)]


def lz_decode(payload: bytes, enc_len, chunk_size: int, n: int, lib=None) -> bytes:
    """lz_decode (codec.hpp:237-244) of lz_encode's output back to n bytes;
    CorruptStreamError like lz_decode_chunk (codec.hpp:177-220)."""
    L = _lib(lib)
    pl = np.frombuffer(bytes(payload) + b"\0", dtype=np.uint8)
    lens = (abi.u64 * max(len(enc_len), 1))(*enc_len)
    out = np.empty(max(n, 1), dtype=np.uint8)
    L.check(L.wg_lz_decode(pl.ctypes.data, lens, chunk_size, out.ctypes.data, n))
    return out[:n].tobytes()


# ---- patchgrid.hpp ---------------------------------------------------------------


@dataclass
class PatchGrid:
    """PatchGrid (patchgrid.hpp:38-55) as one grid buffer: patches x
    components x true (logical + 2) arrays."""

    global_dims: tuple
    splits: tuple
    components: int = 1
    periodic: bool = True
    data: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        self.logical = tuple((g - 1) // s + 1 for g, s in zip(self.global_dims, self.splits))
        self.true_dims = tuple(n + 2 for n in self.logical)
        self.npatch = int(np.prod(self.splits))
        if self.data is None:
            self.data = np.zeros((self.npatch, self.components) + self.true_dims)

    def desc(self) -> abi.GridDesc:
        return abi.grid_desc(self.global_dims, self.splits, self.components, self.periodic)

    def patch_coord(self, p: int):
        return tuple(int(x) for x in np.unravel_index(p, self.splits))

    def origin(self, p: int):  # Patch::origin, patchgrid.hpp:91-95
        return tuple(c * (n - 1) for c, n in zip(self.patch_coord(p), self.logical))

    def logical_view(self):
        sl = (slice(None), slice(None)) + tuple(slice(1, n + 1) for n in self.logical)
        return self.data[sl]


def decompose(global_dims, splits, components: int, periodic: bool = True, lib=None) -> PatchGrid:
    """decompose() (patchgrid.hpp:59-103) with the reference's validation."""
    L = _lib(lib)
    g = abi.grid_desc(global_dims, splits, components, periodic)
    pl = (abi.u64 * 3)()
    npatch, nd = abi.u64(), abi.u64()
    L.check(L.wg_grid_geometry(C.byref(g), pl, C.byref(npatch), C.byref(nd)))
    return PatchGrid(tuple(global_dims), tuple(splits), components, periodic)


def fill(grid: PatchGrid, comp: int, f) -> None:
    """fill() (patchgrid.hpp:106-126): f(global index tuple) -> value."""
    for p in range(grid.npatch):
        o = grid.origin(p)
        for idx in np.ndindex(*grid.logical):
            gi = tuple(a + b for a, b in zip(o, idx))
            grid.data[(p, comp) + tuple(i + 1 for i in idx)] = f(gi)


def sync_ghosts(grid: PatchGrid, lib=None) -> None:
    L = _lib(lib)
    d = grid.desc()
    L.check(L.wg_sync_ghosts(C.byref(d), abi.dptr(grid.data)))


def global_mass(grid: PatchGrid, comp: int, lib=None) -> float:
    L = _lib(lib)
    d = grid.desc()
    out = C.c_double()
    L.check(L.wg_global_mass(C.byref(d), abi.dptr(grid.data), comp, C.byref(out)))
    return out.value


def fv_step(cur: PatchGrid, nxt: PatchGrid, scheme: str, dt: float, dx: float, alpha=0.9, beta=0.9,
            gravity=9.81, lib=None) -> None:
    """fv_step<Flux> over every patch (solver.hpp:207-231)."""
    L = _lib(lib)
    d = cur.desc()
    L.check(L.wg_fv_step(C.byref(d), abi.dptr(cur.data), abi.dptr(nxt.data), abi.scheme_id(scheme),
                         alpha, beta, gravity, dt, dx))


def lbm_step(cur: PatchGrid, nxt: PatchGrid, tau: float, lib=None) -> None:
    L = _lib(lib)
    d = cur.desc()
    L.check(L.wg_lbm_step(C.byref(d), abi.dptr(cur.data), abi.dptr(nxt.data), tau))


# ---- pipeline.hpp ------------------------------------------------------------------

_ROW_FIELDS = ["step", "time", "dense_bytes", "compressed_bytes", "ratio", "nnz", "zeroed", "global_mass", "l2"]


@dataclass
class RunConfig:
    """RunConfig + SimConfig (pipeline.hpp:23-38, solver.hpp:26-46) + LBM knobs."""

    scheme: str = "transport"
    nx: int = 129
    splits: tuple = (2, 2)
    cfl: float = 0.45
    t_end: float = 0.5
    alpha: float = 0.9
    beta: float = 0.9
    gravity: float = 9.81
    domain_length: float = 1.0
    levels: int = 4
    spec: ThresholdSpec = field(default_factory=ThresholdSpec)
    no_compression: bool = False
    strict: bool = False
    threads: int = 1
    compute_l2: bool = True
    lbm_steps: int = 100
    lbm_tau: float = 0.6
    lbm_u0: float = 0.05
    lbm_kappa: float = 80.0
    lbm_delta: float = 0.05
    store_budget_bytes: int = 0
    tile_rows: int = 1
    metrics_path: str = ""       # RunConfig::metrics_path: CSV of the rows (pipeline.hpp:162-166)
    codec: str = "csr"           # RunConfig::codec: "csr" or "lz" (codec.hpp:250)
    chunk_size: int = 64 * 1024  # RunConfig::chunk_size: LZ chunk bytes (pipeline.hpp:28)

    def to_c(self) -> abi.RunConfigC:
        c = abi.RunConfigC()
        c.scheme = abi.scheme_id(self.scheme)
        c.levels = self.levels
        c.nx = self.nx
        c.splits[0], c.splits[1] = self.splits
        c.cfl, c.t_end, c.alpha, c.beta = self.cfl, self.t_end, self.alpha, self.beta
        c.gravity, c.domain_length = self.gravity, self.domain_length
        c.threshold_mode = abi.threshold_mode(self.spec.mode)
        c.codec = {"csr": 1, "lz": 2}[self.codec]
        c.c, c.threshold_alpha = self.spec.c, self.spec.alpha
        c.no_compression = int(self.no_compression)
        c.strict = int(self.strict)
        c.threads = self.threads
        c.compute_l2 = int(self.compute_l2)
        c.lbm_steps = self.lbm_steps
        c.lbm_tau, c.lbm_u0, c.lbm_kappa, c.lbm_delta = self.lbm_tau, self.lbm_u0, self.lbm_kappa, self.lbm_delta
        c.store_budget_bytes = self.store_budget_bytes
        c.tile_rows = self.tile_rows
        c.lz_chunk_size = self.chunk_size
        return c

    @property
    def components(self) -> int:
        return {"transport": 1, "swe": 3}.get(self.scheme, 9)


@dataclass
class RunResult:  # pipeline.hpp:65-70
    rows: list
    summary: dict
    grid: PatchGrid
    t_final: float


def run(cfg: RunConfig, lib=None, max_rows: int = 1 << 17) -> RunResult:
    """run(RunConfig) (pipeline.hpp:129-305)."""
    L = _lib(lib)
    c = cfg.to_c()
    n = abi.u64()
    L.check(L.wg_run_grid_doubles(C.byref(c), C.byref(n)))
    steps = abi.u64()
    L.check(L.wg_run_step_count(C.byref(c), C.byref(steps)))
    cap = steps.value if steps.value else max_rows
    rows = (abi.MetricsRowC * max(cap, 1))()
    nr = abi.u64()
    grid = PatchGrid((cfg.nx, cfg.nx), tuple(cfg.splits), cfg.components, True)
    assert grid.data.size == n.value
    s = abi.RunSummaryC()
    L.check(L.wg_run(C.byref(c), rows, cap, C.byref(nr), abi.dptr(grid.data), C.byref(s)))
    out_rows = [{k: getattr(r, k) for k in _ROW_FIELDS} for r in rows[: min(nr.value, cap)]]
    summary = {k: getattr(s, k) for k, _ in abi.RunSummaryC._fields_}
    if cfg.metrics_path:
        write_metrics_csv(out_rows, cfg.metrics_path)
    return RunResult(out_rows, summary, grid, s.t_final)


METRICS_HEADER = "step,time,dense_bytes,compressed_bytes,ratio,nnz,zeroed,global_mass,l2_error\n"


def metrics_csv_row(r: dict) -> str:
    """write_metrics_row (pipeline.hpp:78-84): %zu for counts, %.17g for reals."""
    return "%d,%.17g,%d,%d,%.17g,%d,%d,%.17g,%.17g\n" % (
        r["step"], r["time"], r["dense_bytes"], r["compressed_bytes"], r["ratio"], r["nnz"], r["zeroed"],
        r["global_mass"], r["l2"])


def write_metrics_csv(rows, path) -> None:
    """The metrics file of run() (write_metrics_header/row, pipeline.hpp:74-84)."""
    with open(path, "w") as f:
        f.write(METRICS_HEADER)
        for r in rows:
            f.write(metrics_csv_row(r))


def initial_state(cfg: RunConfig, lib=None) -> PatchGrid:
    L = _lib(lib)
    c = cfg.to_c()
    grid = PatchGrid((cfg.nx, cfg.nx), tuple(cfg.splits), cfg.components, True)
    L.check(L.wg_run_initial_state(C.byref(c), abi.dptr(grid.data)))
    return grid
