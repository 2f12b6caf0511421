"""Patch-row sharding of the compressed stencil loop over GPUs.

One process per GPU.  Rank r owns a contiguous range of patch rows (a patch
row lies wholly on one rank, so the dim-1 ghost sync and the corner fill stay
local).  After every step the only exchange is the ring of halo lines:
rank r sends logical row 1 of its first patch row to r-1 and logical row n-2
of its last patch row to r+1 (periodic ring), i.e. exactly the values that
sync_ghosts (patchgrid.hpp:131-201) copies across the rank boundary.
Reductions (mass, nnz, zeroed, bytes) are all-reduced once, at the end.
The shallow-water scheme adds one collective per step: its CFL time step is a
max over the whole grid (cfl_dt, solver.hpp:242-258), so every rank's max
wave speed is all-reduced with MAX before the next step (8 bytes; the session
computes dt from it on the device).

The exchange uses torch.distributed point-to-point (NCCL over NVLink on GPU,
gloo on CPU in the tests) on tensors that alias the session's halo blocks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi


def shard_rows(nrows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced patch-row range of `rank` (row-major patches,
    patchgrid.hpp:50-54, so a shard is a contiguous patch-index range)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if nrows < world:
        raise ValueError(f"{nrows} patch rows cannot be split over {world} ranks")
    base, extra = divmod(nrows, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def ring_neighbours(rank: int, world: int) -> tuple[int, int]:
    """(above, below) in the periodic ring of patch-row shards."""
    return (rank - 1) % world, (rank + 1) % world


def exchange_halos(send_lo, send_hi, recv_lo, recv_hi, rank: int, world: int, dist) -> None:
    """Ring exchange of halo blocks.  recv_lo <- above.send_hi,
    recv_hi <- below.send_lo.  Operations are posted in one fixed order on
    every rank so that world == 2 (above == below) still pairs correctly."""
    above, below = ring_neighbours(rank, world)
    staged = send_lo.is_cuda and dist.get_backend() == "gloo"  # gloo moves host tensors only
    if staged:
        dev = (recv_lo, recv_hi)
        send_lo, send_hi = send_lo.cpu(), send_hi.cpu()
        recv_lo, recv_hi = torch_empty_like_cpu(recv_lo), torch_empty_like_cpu(recv_hi)
    ops = [
        dist.P2POp(dist.isend, send_hi, below),
        dist.P2POp(dist.isend, send_lo, above),
        dist.P2POp(dist.irecv, recv_lo, above),
        dist.P2POp(dist.irecv, recv_hi, below),
    ]
    # NCCL: wait() orders the session stream after the transfer (a device-side
    # dependency, no host wait); gloo (tests on one GPU) completes on the host
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if staged:
        dev[0].copy_(recv_lo)
        dev[1].copy_(recv_hi)


def torch_empty_like_cpu(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype, device="cpu")


def collective_device(dist, device):
    """Where collective operands live: the GPU for NCCL, the host for gloo
    (the multi-process path run on one GPU in tests/test_gpu_multiproc.py)."""
    return "cpu" if dist.get_backend() == "gloo" else device


class _DevArray:
    """A raw device pointer exposed through __cuda_array_interface__ so that
    torch.as_tensor aliases it without a copy."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def reduce_rows(rows: list[dict], dist, device) -> list[dict]:
    """All-reduce per-shard metrics rows into whole-grid rows (sums; ratio
    recomputed as in pipeline.hpp:270-272)."""
    import torch

    keys = ["dense_bytes", "compressed_bytes", "nnz", "zeroed"]
    device = collective_device(dist, device)
    ints = torch.tensor([[r[k] for k in keys] for r in rows], dtype=torch.int64, device=device)
    # global_mass and the transport l2 are sums over patches: each shard's
    # share adds exactly (l2_scale is applied per shard, solver.hpp:302-304)
    dbl = torch.tensor([[r["global_mass"], r.get("l2", 0.0)] for r in rows], dtype=torch.float64, device=device)
    dist.all_reduce(ints)
    dist.all_reduce(dbl)
    out = []
    for r, iv, (m, l2) in zip(rows, ints.tolist(), dbl.tolist()):
        o = dict(r)
        o.update(dict(zip(keys, iv)))
        o["global_mass"] = m
        if "l2" in r:
            o["l2"] = l2
        o["ratio"] = o["dense_bytes"] / o["compressed_bytes"] if o["compressed_bytes"] > 0 else 1.0
        out.append(o)
    return out


@dataclass
class ShardInfo:
    rank: int
    world: int
    row_begin: int
    row_end: int
    device: int


class ShardedSession:
    """A device session over this rank's patch rows, stepping in lock-step
    with the other ranks."""

    def __init__(self, lib: abi.Lib, cfg, shard: ShardInfo, stream_ptr: int | None, dist=None):
        self.lib, self.cfg, self.shard, self.dist = lib, cfg, shard, dist
        c = cfg.to_c()
        sh = abi.ShardC()
        sh.rank, sh.world, sh.device = shard.rank, shard.world, shard.device
        sh.row_begin, sh.row_end = shard.row_begin, shard.row_end
        self.handle = abi.vp()
        lib.check(lib.wg_session_create(C.byref(c), C.byref(sh), abi.vp(stream_ptr) if stream_ptr else None,
                                        C.byref(self.handle)))
        self.info = abi.SessionInfoC()
        lib.check(lib.wg_session_info_get(self.handle, C.byref(self.info)))
        self._halo = None
        self.swe = cfg.scheme == "swe"
        self.peer = False
        self._ipc_opened: list[int] = []

    # ---- peer halo mode (wg_session_peer_*): the step kernels store the halo
    # lines into the neighbours' halo slots over NVLink, no exchange between
    # steps.  Transport and D2Q9; opt-in (bench: WG_PEER_HALOS=1).
    def peer_export(self) -> dict:
        m0, m1, fl, rows = abi.vp(), abi.vp(), abi.vp(), C.c_uint32()
        self.lib.check(self.lib.wg_session_peer_export(self.handle, C.byref(m0), C.byref(m1), C.byref(fl),
                                                       C.byref(rows)))
        return {"mem0": m0.value, "mem1": m1.value, "flags": fl.value, "rows": rows.value}

    def peer_attach(self, above: dict, below: dict):
        self.lib.check(self.lib.wg_session_peer_attach(
            self.handle, abi.vp(above["mem0"]), abi.vp(above["mem1"]), abi.vp(above["flags"]), above["rows"],
            abi.vp(below["mem0"]), abi.vp(below["mem1"]), abi.vp(below["flags"]), below["rows"]))
        self.peer = True

    def peer_push(self):
        self.lib.check(self.lib.wg_session_peer_push(self.handle))

    def connect_peers(self):
        """Multi-process: map the ring neighbours' edge allocations and flag
        words by CUDA IPC (handles all-gathered over the process group) and
        attach them.  Collective: every rank calls it."""
        exp = self.peer_export()
        mine = {"rows": exp["rows"]}
        for k in ("mem0", "mem1", "flags"):
            buf = C.create_string_buffer(64)
            self.lib.check(self.lib.wg_ipc_handle(abi.vp(exp[k]), buf))
            mine[k] = buf.raw
        allx = [None] * self.shard.world
        self.dist.all_gather_object(allx, mine)
        above_r, below_r = ring_neighbours(self.shard.rank, self.shard.world)
        opened: dict[int, dict] = {}
        for r in {above_r, below_r}:
            d = {"rows": allx[r]["rows"]}
            for k in ("mem0", "mem1", "flags"):
                p = abi.vp()
                self.lib.check(self.lib.wg_ipc_open(allx[r][k], C.byref(p)))
                self._ipc_opened.append(p.value)
                d[k] = p.value
            opened[r] = d
        self.peer_attach(opened[above_r], opened[below_r])

    def close(self):
        if self.handle:
            self.lib.wg_session_destroy(self.handle)
            self.handle = abi.vp()
        for p in self._ipc_opened:
            self.lib.wg_ipc_close(abi.vp(p))
        self._ipc_opened = []

    def upload(self, host_grid: np.ndarray):
        self.lib.check(self.lib.wg_session_upload(self.handle, abi.dptr(host_grid)))
        self._initial_exchange()

    def step_host(self, host_grid: np.ndarray, dt: float = 1.0):
        """Step 1 straight from a host initial state (wg_session_step_host:
        the raw state streams through the device and never enters the store;
        one-shard D2Q9, C4)."""
        if self.shard.world != 1:
            raise ValueError("step_host: one-shard sessions only")
        self.lib.check(self.lib.wg_session_step_host(self.handle, abi.dptr(host_grid), dt))

    def download(self, host_grid: np.ndarray):
        """The decoded state of this shard into a host grid buffer."""
        self.lib.check(self.lib.wg_session_download(self.handle, abi.dptr(host_grid)))

    def init_device(self):
        """Initial state generated and compressed on the device (C4/C5)."""
        self.lib.check(self.lib.wg_session_init_device(self.handle))
        self._initial_exchange()

    def _initial_exchange(self):
        """After upload / init / load: the edges were rebuilt locally."""
        if self.peer:
            if self.dist is not None:
                self.dist.barrier()  # every neighbour rebuilt its own edges first
            self.peer_push()
        else:
            self._exchange()

    def _exchange(self):
        if self.shard.world > 1 and not self.peer:
            s_lo, s_hi, r_lo, r_hi = self.halo_tensors()
            exchange_halos(s_lo, s_hi, r_lo, r_hi, self.shard.rank, self.shard.world, self.dist)
            if self.swe:
                v = self.cfl_vmax_tensor()
                if self.dist.get_backend() == "gloo":
                    h = v.cpu()
                    self.dist.all_reduce(h, op=self.dist.ReduceOp.MAX)
                    v.copy_(h)
                else:
                    self.dist.all_reduce(v, op=self.dist.ReduceOp.MAX)

    def cfl_vmax_tensor(self):
        """SWE: the next step's max wave speed (int64 view of the non-negative
        double's bits, so MAX over int64 is MAX over the doubles)."""
        import torch

        p = abi.vp()
        self.lib.check(self.lib.wg_session_cfl_vmax(self.handle, C.byref(p)))
        arr = _DevArray(p.value, 1)
        arr.__cuda_array_interface__["typestr"] = "<i8"
        return torch.as_tensor(arr, device=f"cuda:{self.shard.device}")

    def halo_tensors(self):
        import torch

        ptrs = [abi.vp() for _ in range(4)]
        self.lib.check(self.lib.wg_session_halo(self.handle, *[C.byref(p) for p in ptrs]))
        n = self.info.halo_doubles
        return [torch.as_tensor(_DevArray(p.value, n), device=f"cuda:{self.shard.device}") for p in ptrs]

    def save(self, path: str):
        """Checkpoint this shard's compressed store (WGS1 + WGC1 records)."""
        self.lib.check(self.lib.wg_session_save(self.handle, str(path).encode()))

    def load(self, path: str):
        """Resume from a checkpoint written by save() for the same shard."""
        self.lib.check(self.lib.wg_session_load(self.handle, str(path).encode()))
        self._initial_exchange()

    def step(self, dt: float = 1.0):
        self.lib.check(self.lib.wg_session_step(self.handle, dt))
        self._exchange()  # the halo blocks move with the double buffer: re-fetched every step (host mode)

    def sync(self):
        self.lib.check(self.lib.wg_session_sync(self.handle))

    def rows(self) -> list[dict]:
        n = abi.u64()
        self.lib.check(self.lib.wg_session_metrics(self.handle, None, 0, C.byref(n)))
        buf = (abi.MetricsRowC * max(n.value, 1))()
        self.lib.check(self.lib.wg_session_metrics(self.handle, buf, n.value, C.byref(n)))
        keys = [k for k, _ in abi.MetricsRowC._fields_]
        return [{k: getattr(r, k) for k in keys} for r in buf[: n.value]]

    def last_row(self) -> dict:
        r = abi.MetricsRowC()
        self.lib.check(self.lib.wg_session_last_row(self.handle, C.byref(r)))
        return {k: getattr(r, k) for k, _ in abi.MetricsRowC._fields_}
