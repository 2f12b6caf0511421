"""CPU, world_size 2 (gloo): the N>1 path of the sharded loop.

The shard logic of paper_2302_09883_b200/distributed.py (patch-row ranges,
the periodic halo ring, the metric all-reduce) is exercised with a stand-in
for the device session whose per-shard step is the C oracle on that shard's
patch rows plus the two halo rows.  The N-shard state must equal the 1-shard
oracle run bit for bit (the exchange is a pure copy)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2302_09883_b200 import api
from paper_2302_09883_b200.distributed import exchange_halos, reduce_rows, ring_neighbours, shard_rows


def test_shard_rows_cover_and_balance():
    for nrows in (2, 5, 16, 1024):
        for world in (1, 2, 3, 8):
            if world > nrows:
                with pytest.raises(ValueError):
                    shard_rows(nrows, 0, world)
                continue
            parts = [shard_rows(nrows, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == nrows
            assert all(parts[k][1] == parts[k + 1][0] for k in range(world - 1))
            sizes = [e - b for b, e in parts]
            assert max(sizes) - min(sizes) <= 1
    assert ring_neighbours(0, 4) == (3, 1) and ring_neighbours(3, 4) == (2, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_kw, steps, out):
    import torch.distributed as dist
    import torch

    from tests.conftest import ORACLE_C
    from paper_2302_09883_b200 import abi

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle = abi.Lib(ORACLE_C)
    cfg = api.RunConfig(**cfg_kw)
    full = api.initial_state(cfg, lib=oracle)
    P0, P1 = cfg.splits
    n = full.logical[0]
    rb, re_ = shard_rows(P0, rank, world)
    R = re_ - rb
    tp = n + 2
    # this shard's patches (R rows) plus one halo patch row above and below
    own = full.data.reshape(P0, P1, full.components, tp, tp)[rb:re_].copy()
    dt = cfg.cfl * (1.0 / (cfg.nx - 1)) / max(cfg.alpha, cfg.beta)
    for _ in range(steps):
        # halo blocks: logical row 1 of the first patch row / row n-2 of the last
        send_lo = torch.from_numpy(np.ascontiguousarray(own[0, :, :, 2, 1:-1]))
        send_hi = torch.from_numpy(np.ascontiguousarray(own[R - 1, :, :, n - 1, 1:-1]))
        recv_lo = torch.empty_like(send_hi)
        recv_hi = torch.empty_like(send_lo)
        exchange_halos(send_lo, send_hi, recv_lo, recv_hi, rank, world, dist)
        # assemble a periodic-in-dim-1, halo-padded local grid: R+2 patch rows
        loc = np.zeros((R + 2, P1, full.components, tp, tp))
        loc[1:R + 1] = own
        loc[0, :, :, n - 1, 1:-1] = recv_lo.numpy()  # the row above's logical n-2 line
        loc[R + 1, :, :, 2, 1:-1] = recv_hi.numpy()  # the row below's logical 1 line
        g = api.PatchGrid(((R + 2) * (n - 1) + 1, cfg.nx), (R + 2, P1), full.components, True,
                          data=loc.reshape(-1, full.components, tp, tp).copy())
        api.sync_ghosts(g, lib=oracle)  # dim-0 ghosts of the owned rows now come from the halo rows
        nxt = api.PatchGrid(g.global_dims, g.splits, g.components, True, data=g.data.copy())
        api.fv_step(g, nxt, "transport", dt, 1.0 / (cfg.nx - 1), lib=oracle)
        own = nxt.data.reshape(R + 2, P1, full.components, tp, tp)[1:R + 1].copy()
    rows = [{"dense_bytes": R * P1, "compressed_bytes": rank + 1, "nnz": 10 * rank, "zeroed": 1,
             "global_mass": float(own[:, :, 0, 1:-1, 1:-1].sum()), "ratio": 0.0}]
    red = reduce_rows(rows, dist, "cpu")
    out.put((rank, own, red))
    dist.destroy_process_group()


def test_two_rank_halo_ring_equals_single_shard(oracle):
    import multiprocessing as mp

    cfg_kw = dict(scheme="transport", nx=65, splits=(4, 4), levels=3, spec=api.ThresholdSpec("capped", 0.0))
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg_kw, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in procs:
        rank, own, red = q.get(timeout=120)
        res[rank] = (own, red)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-shard reference: the same FV steps on the whole periodic grid
    cfg = api.RunConfig(**cfg_kw)
    g = api.initial_state(cfg, lib=oracle)
    dt = cfg.cfl * (1.0 / 64) / 0.9
    for _ in range(steps):
        api.sync_ghosts(g, lib=oracle)
        nxt = api.PatchGrid(g.global_dims, g.splits, 1, True, data=g.data.copy())
        api.fv_step(g, nxt, "transport", dt, 1.0 / 64, lib=oracle)
        g = nxt
    whole = g.data.reshape(4, 4, 1, 19, 19)
    got = np.concatenate([res[0][0], res[1][0]], axis=0)
    lv = (slice(None), slice(None), slice(None), slice(1, -1), slice(1, -1))
    assert np.array_equal(got[lv].view(np.uint64), whole[lv].view(np.uint64))
    # all-reduced metrics: integer sums exact, ratio recomputed
    red0, red1 = res[0][1][0], res[1][1][0]
    assert red0 == red1
    assert red0["compressed_bytes"] == 3 and red0["nnz"] == 10 and red0["dense_bytes"] == 16
    assert red0["ratio"] == 16 / 3
