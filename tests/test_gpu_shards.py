"""The sharded device path on ONE GPU: `world` patch-row shards
as `world` sessions of one process, stepped in lock-step on one stream, with
the halo ring (and the SWE CFL max) exchanged by device copies between
steps — exactly the data movement distributed.ShardedSession does over NCCL,
minus the transport.  No kernel waits on another shard's kernel.

The N-shard state must be bitwise equal to the 1-shard state (the exchange
is a pure copy; SURVEY §8e "Test"), and the per-shard metrics must sum to
the 1-shard metrics (integer counts exactly, mass to round-off)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api
from paper_2302_09883_b200.distributed import ShardInfo, ShardedSession, shard_rows

from .test_gpu_session import bits

pytestmark = pytest.mark.gpu


class LocalShards:
    def __init__(self, lib, cfg: api.RunConfig, world: int):
        import torch

        self.torch = torch
        self.lib, self.cfg, self.world = lib, cfg, world
        self.stream = torch.cuda.Stream()
        P0 = cfg.splits[0] * max(cfg.tile_rows, 1)
        self.ranges = [shard_rows(P0, r, world) for r in range(world)]
        self.sessions = [ShardedSession(lib, cfg, ShardInfo(r, world, rb, re_, 0), self.stream.cuda_stream, None)
                         for r, (rb, re_) in enumerate(self.ranges)]

    def close(self):
        for s in self.sessions:
            s.close()

    def upload(self, grid: api.PatchGrid):
        P1 = self.cfg.splits[1]
        per = grid.data.size // grid.data.shape[0]
        flat = grid.data.reshape(grid.data.shape[0], per)
        self._keep = []
        for s, (rb, re_) in zip(self.sessions, self.ranges):
            part = np.ascontiguousarray(flat[rb * P1: re_ * P1]).reshape(-1)
            self._keep.append(part)
            self.lib.check(self.lib.wg_session_upload(s.handle, abi.dptr(part)))
        self.exchange()

    def exchange(self):
        torch = self.torch
        halos = [s.halo_tensors() for s in self.sessions]
        with torch.cuda.stream(self.stream):
            for r in range(self.world):
                above, below = (r - 1) % self.world, (r + 1) % self.world
                halos[r][2].copy_(halos[above][1])  # recv_lo <- above.send_hi
                halos[r][3].copy_(halos[below][0])  # recv_hi <- below.send_lo
            if self.cfg.scheme == "swe":
                v = [s.cfl_vmax_tensor() for s in self.sessions]
                m = torch.stack(v).max()
                for t in v:
                    t.copy_(m)

    def step(self):
        for s in self.sessions:
            self.lib.check(self.lib.wg_session_step(s.handle, 1.0))
        self.exchange()

    def download(self) -> np.ndarray:
        self.stream.synchronize()
        parts = []
        for s in self.sessions:
            n = s.info.npatch_local * s.info.components * (s.info.patch_n + 2) ** 2
            out = np.zeros(n)
            self.lib.check(self.lib.wg_session_download(s.handle, abi.dptr(out)))
            parts.append(out)
        return np.concatenate(parts)

    def rows(self):
        per = [s.rows() for s in self.sessions]
        assert len({len(p) for p in per}) == 1
        return per


def _cfg(scheme, nx, splits, levels, c, **kw):
    cfg = api.RunConfig(scheme=scheme, nx=nx, splits=splits, levels=levels,
                        spec=api.ThresholdSpec("capped" if scheme != "swe" else "constant", c), compute_l2=False,
                        **kw)
    if scheme == "transport":
        cfg.t_end = 1.0
    return cfg


@pytest.mark.parametrize(
    "scheme,nx,splits,levels,c,world,steps",
    [("transport", 257, (8, 8), 4, 1e-3, 2, 6),
     ("transport", 257, (8, 8), 4, 1e-3, 3, 6),   # uneven shards (3, 3, 2 rows)
     ("lbm", 257, (8, 8), 4, 1e-3, 2, 5),
     ("lbm", 129, (4, 4), 4, 1e-3, 4, 5),          # one patch row per shard
     ("swe", 129, (4, 4), 4, 5e-4, 2, 8),
     ("swe", 257, (4, 4), 4, 5e-4, 4, 6)],         # one patch row per shard, CFL max all-reduced
)
def test_shards_equal_single(product, scheme, nx, splits, levels, c, world, steps):
    cfg = _cfg(scheme, nx, splits, levels, c, t_end=1.0) if scheme == "swe" else _cfg(scheme, nx, splits, levels, c)
    g0 = api.initial_state(cfg, lib=product)
    single = LocalShards(product, cfg, 1)
    multi = LocalShards(product, cfg, world)
    try:
        single.upload(g0)
        multi.upload(g0)
        dt = cfg.cfl / (nx - 1) / 0.9
        for _ in range(steps):
            for s in single.sessions:
                product.check(product.wg_session_step(s.handle, dt))
            single.exchange()
            for s in multi.sessions:
                product.check(product.wg_session_step(s.handle, dt))
            multi.exchange()
        a, b = single.download(), multi.download()
        assert np.array_equal(bits(a), bits(b)), f"{np.sum(a != b)} values differ"
        r1 = single.rows()[0]
        rn = multi.rows()
        assert len(r1) == steps
        for k in range(steps):
            for key in ("step", "dense_bytes", "compressed_bytes", "nnz", "zeroed"):
                assert r1[k][key] == (rn[0][k][key] if key == "step" else sum(p[k][key] for p in rn)), key
            assert all(p[k]["time"] == r1[k]["time"] for p in rn)
            m = sum(p[k]["global_mass"] for p in rn)
            assert abs(m - r1[k]["global_mass"]) <= 1e-12 * abs(r1[k]["global_mass"])
    finally:
        single.close()
        multi.close()


def test_swe_single_shard_session_matches_run(product, oracle_sq):
    """The single-shard path above is the product's own run(): cross-check
    one SWE case against the oracle end to end."""
    cfg = _cfg("swe", 129, (4, 4), 4, 5e-4, t_end=0.002)
    ref = api.run(cfg, lib=oracle_sq)
    g0 = api.initial_state(cfg, lib=product)
    one = LocalShards(product, cfg, 1)
    try:
        one.upload(g0)
        for _ in range(len(ref.rows) + 2):
            one.step()
        a = one.download().reshape(ref.grid.data.shape)
        la = a[(slice(None), slice(None)) + tuple(slice(1, n + 1) for n in ref.grid.logical)]
        assert np.array_equal(bits(la), bits(ref.grid.logical_view()))
    finally:
        one.close()


class PeerShards(LocalShards):
    """The same shards in peer halo mode: each session is attached to its
    ring neighbours' edge allocations (plain device pointers here: one
    process; CUDA IPC across processes), the step kernels store the halo
    lines into the neighbours' halo slots themselves and the sessions
    synchronise through the device flag words — no exchange between steps.
    All shards run in order on one stream, so every device-side wait is
    already satisfied when it is reached (no kernel waits on a kernel that
    has not run)."""

    def __init__(self, lib, cfg, world):
        super().__init__(lib, cfg, world)
        ex = [s.peer_export() for s in self.sessions]
        for r, s in enumerate(self.sessions):
            s.peer_attach(ex[(r - 1) % world], ex[(r + 1) % world])

    def exchange(self):
        pass  # the step kernels did it

    def upload(self, grid: api.PatchGrid):
        P1 = self.cfg.splits[1]
        per = grid.data.size // grid.data.shape[0]
        flat = grid.data.reshape(grid.data.shape[0], per)
        self._keep = []
        for s, (rb, re_) in zip(self.sessions, self.ranges):
            part = np.ascontiguousarray(flat[rb * P1: re_ * P1]).reshape(-1)
            self._keep.append(part)
            self.lib.check(self.lib.wg_session_upload(s.handle, abi.dptr(part)))
        for s in self.sessions:  # every shard built its own edges: now the halo rows
            s.peer_push()


@pytest.mark.parametrize(
    "scheme,nx,splits,levels,c,world,steps,codec",
    [("transport", 257, (8, 8), 4, 1e-3, 2, 6, "csr"),
     ("transport", 257, (8, 8), 4, 1e-3, 3, 6, "csr"),   # uneven shards
     ("lbm", 257, (8, 8), 4, 1e-3, 2, 5, "csr"),
     ("lbm", 129, (4, 4), 4, 1e-3, 4, 5, "csr"),          # one patch row per shard
     ("lbm", 129, (4, 4), 4, 1e-3, 2, 4, "lz")],
)
def test_peer_halos_equal_single(product, scheme, nx, splits, levels, c, world, steps, codec):
    cfg = _cfg(scheme, nx, splits, levels, c, codec=codec)
    g0 = api.initial_state(cfg, lib=product)
    single = LocalShards(product, cfg, 1)
    multi = PeerShards(product, cfg, world)
    try:
        single.upload(g0)
        multi.upload(g0)
        dt = cfg.cfl / (nx - 1) / 0.9
        for _ in range(steps):
            for s in single.sessions:
                product.check(product.wg_session_step(s.handle, dt))
            single.exchange()
            for s in multi.sessions:
                product.check(product.wg_session_step(s.handle, dt))
        a, b = single.download(), multi.download()
        for s in multi.sessions:
            s.sync()  # device error word (a peer wait that timed out raises here)
        assert np.array_equal(bits(a), bits(b)), f"{np.sum(a != b)} values differ"
        r1, rn = single.rows()[0], multi.rows()
        for k in range(steps):
            for key in ("dense_bytes", "compressed_bytes", "nnz", "zeroed"):
                assert r1[k][key] == sum(p[k][key] for p in rn), key
    finally:
        single.close()
        multi.close()


def test_peer_halos_reject_swe(product):
    cfg = _cfg("swe", 129, (4, 4), 4, 5e-4, t_end=1.0)
    two = LocalShards(product, cfg, 2)
    try:
        ex = [s.peer_export() for s in two.sessions]
        with pytest.raises(ValueError):
            two.sessions[0].peer_attach(ex[1], ex[1])
    finally:
        two.close()


def _block(lib, sess, patch: int, comp: int, n: int):
    v = np.zeros(n * n)
    col = np.zeros(n * n, dtype=np.uint32)
    row = np.zeros(n + 1, dtype=np.uint32)
    nnz, raw = abi.u64(), C.c_int32()
    lib.check(lib.wg_session_patch_csr(sess.handle, patch, comp, abi.dptr(v), col.ctypes.data_as(C.POINTER(C.c_uint32)),
                                       row.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(nnz), C.byref(raw)))
    k = nnz.value if not raw.value else n * n
    return raw.value, bits(v[:k]).tobytes(), col[: nnz.value].tobytes(), row.tobytes()


def test_peer_halos_c5_geometry(product):
    """Peer halo mode at the C5 geometry (65536^2 grid: 1024 x 1024 patches of
    65^2 points, L = 4, capped 1e-3, device initial state): a band of 8 patch
    rows (8192 patches) as ONE shard (periodic over the band) against the
    same band as 4 peer-attached shards of 2 rows each — the step kernels
    store every halo line into the neighbour shard's slots.  Per-step counts
    equal, masses to round-off, and the stored CSR blocks of sampled patches
    (both sides of every shard boundary) bitwise equal."""
    import torch

    cfg = _cfg("lbm", 65537, (1024, 1024), 4, 1e-3)
    R, world, steps, n = 8, 4, 4, 65
    stream = torch.cuda.Stream()
    single = ShardedSession(product, cfg, ShardInfo(0, 1, 0, R, 0), stream.cuda_stream, None)
    per = R // world
    multi = [ShardedSession(product, cfg, ShardInfo(r, world, per * r, per * (r + 1), 0), stream.cuda_stream, None)
             for r in range(world)]
    try:
        ex = [s.peer_export() for s in multi]
        for r, s in enumerate(multi):
            s.peer_attach(ex[(r - 1) % world], ex[(r + 1) % world])
        product.check(product.wg_session_init_device(single.handle))
        for s in multi:
            product.check(product.wg_session_init_device(s.handle))
        for s in multi:  # every shard built its own edges: now the halo rows
            s.peer_push()
        for _ in range(steps):
            product.check(product.wg_session_step(single.handle, 1.0))
            for s in multi:
                product.check(product.wg_session_step(s.handle, 1.0))
        single.sync()
        for s in multi:
            s.sync()
        r1, rn = single.rows(), [s.rows() for s in multi]
        assert len(r1) == steps
        for k in range(steps):
            for key in ("dense_bytes", "compressed_bytes", "nnz", "zeroed"):
                assert r1[k][key] == sum(p[k][key] for p in rn), key
            m = sum(p[k]["global_mass"] for p in rn)
            assert abs(m - r1[k]["global_mass"]) <= 1e-12 * abs(r1[k]["global_mass"])
        P1 = 1024
        for row in range(R):  # first, middle and last patch of every patch row, all 9 populations
            owner, local_row = row // per, row % per
            for col in (0, 511, 1023):
                for q in range(9):
                    a = _block(product, single, row * P1 + col, q, n)
                    b = _block(product, multi[owner], local_row * P1 + col, q, n)
                    assert a == b, (row, col, q)
    finally:
        single.close()
        for s in multi:
            s.close()


def test_shards_transport_l2_sums(product):
    """compute_l2 on (run()'s default): every shard reports its share of the
    l2_error sum of the global grid (l2_scale per shard, solver.hpp:302-304);
    the shares add up to the one-shard value (distributed.reduce_rows sums
    them across ranks)."""
    cfg = _cfg("transport", 257, (8, 8), 4, 1e-3)
    cfg.compute_l2 = True
    g0 = api.initial_state(cfg, lib=product)
    single = LocalShards(product, cfg, 1)
    multi = LocalShards(product, cfg, 3)
    try:
        single.upload(g0)
        multi.upload(g0)
        dt = cfg.cfl / (cfg.nx - 1) / 0.9
        for _ in range(4):
            for sh in (single, multi):
                for s in sh.sessions:
                    product.check(product.wg_session_step(s.handle, dt))
                sh.exchange()
        r1, rn = single.rows()[0], multi.rows()
        for k in range(4):
            total = sum(p[k]["l2"] for p in rn)
            assert r1[k]["l2"] > 0.0
            assert abs(total - r1[k]["l2"]) <= 1e-12 * r1[k]["l2"], (k, total, r1[k]["l2"])
    finally:
        single.close()
        multi.close()


def test_c5_full_size_two_shards_equal_one(product):
    """C5 at its full size (65536^2: 1024 x 1024 patches of 65^2, L = 4,
    capped 1e-3, store budget 24 GiB per shard, device-generated initial
    state): the grid as 2 patch-row shards with the halo ring exchanged
    between steps equals the one-shard run — every metrics row (the shards'
    integer counts summed exactly, masses to round-off), the stored blocks of
    sampled patches on both sides of both shard boundaries bitwise; mass
    conserved and every block at the L = 4 floor."""
    cfg = _cfg("lbm", 65537, (1024, 1024), 4, 1e-3)
    cfg.store_budget_bytes = 24 << 30
    steps, n, P1 = 3, 65, 1024
    single = LocalShards(product, cfg, 1)
    try:
        for s in single.sessions:
            product.check(product.wg_session_init_device(s.handle))
        single.exchange()
        for _ in range(steps):
            single.step()
        single.stream.synchronize()
        r1 = single.rows()[0]
        picks = [(row, col) for row in (0, 511, 512, 1023) for col in (0, 700)]
        want = {(row, col, q): _block(product, single.sessions[0], row * P1 + col, q, n)
                for row, col in picks for q in range(9)}
    finally:
        single.close()
    multi = LocalShards(product, cfg, 2)
    try:
        for s in multi.sessions:
            product.check(product.wg_session_init_device(s.handle))
        multi.exchange()
        for _ in range(steps):
            multi.step()
        multi.stream.synchronize()
        rn = multi.rows()
        for k in range(steps):
            for key in ("dense_bytes", "compressed_bytes", "nnz", "zeroed"):
                assert r1[k][key] == sum(p[k][key] for p in rn), key
            m = sum(p[k]["global_mass"] for p in rn)
            assert abs(m - r1[k]["global_mass"]) <= 1e-12 * abs(r1[k]["global_mass"])
            assert r1[k]["compressed_bytes"] == 1024 * 1024 * 9 * 564
            assert abs(r1[k]["global_mass"] - r1[0]["global_mass"]) <= 1e-12 * abs(r1[0]["global_mass"])
        for row, col in picks:
            sh = 0 if row < 512 else 1
            for q in range(9):
                got = _block(product, multi.sessions[sh], (row - 512 * sh) * P1 + col, q, n)
                assert got == want[(row, col, q)], (row, col, q)
    finally:
        multi.close()
