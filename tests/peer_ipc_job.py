"""One rank of the peer-halo-mode check across PROCESSES (run by
tests/test_gpu_multiproc.py under torchrun, 2 ranks on the one GPU, gloo):
CUDA IPC handles all-gathered over the process group, neighbours' edge
allocations opened and attached (ShardedSession.connect_peers), halo rows
pushed, then lock-step steps whose halo lines the step kernels store into
the other process's memory.  Every step is followed by a stream sync and a
barrier, so each device-side wait is already satisfied when it is reached:
no kernel ever waits on a kernel of the other process.  Rank 0 compares
the assembled 2-shard state with a 1-shard run, bit for bit."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2302_09883_b200 import abi, api  # noqa: E402
from paper_2302_09883_b200.distributed import ShardInfo, ShardedSession, shard_rows  # noqa: E402


def download(lib, s) -> np.ndarray:
    n = s.info.npatch_local * s.info.components * (s.info.patch_n + 2) ** 2
    out = np.zeros(n)
    lib.check(lib.wg_session_download(s.handle, abi.dptr(out)))
    return out


def main():
    scheme, steps = sys.argv[1], int(sys.argv[2])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    lib = abi.Lib(abi.PRODUCT_LIB)
    nx, splits = 257, (8, 8)
    cfg = api.RunConfig(scheme=scheme, nx=nx, splits=splits, levels=4, spec=api.ThresholdSpec("capped", 1e-3),
                        compute_l2=False)
    if scheme == "transport":
        cfg.t_end = 1.0
    g0 = api.initial_state(cfg, lib=lib)
    flat = g0.data.reshape(g0.data.shape[0], -1)
    stream = torch.cuda.Stream()
    rb, re_ = shard_rows(splits[0], rank, world)
    sess = ShardedSession(lib, cfg, ShardInfo(rank, world, rb, re_, 0), stream.cuda_stream, dist)
    dt = cfg.cfl / (nx - 1) / 0.9
    try:
        sess.connect_peers()
        sess.upload(np.ascontiguousarray(flat[rb * splits[1]: re_ * splits[1]]).reshape(-1))
        stream.synchronize()
        dist.barrier()  # both pushes done before any step waits on them
        for _ in range(steps):
            sess.step(dt)
            stream.synchronize()
            dist.barrier()
        sess.sync()
        part = download(lib, sess)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        if rank == 0:
            one = ShardedSession(lib, cfg, ShardInfo(0, 1, 0, splits[0], 0), stream.cuda_stream, None)
            try:
                one.upload(np.ascontiguousarray(flat).reshape(-1))
                for _ in range(steps):
                    one.step(dt)
                ref = download(lib, one)
            finally:
                one.close()
            got = np.concatenate(parts)
            print(json.dumps({"equal": bool(np.array_equal(got.view(np.uint64), ref.view(np.uint64))),
                              "differ": int(np.sum(got != ref)), "peer": sess.peer}))
        dist.barrier()
    finally:
        sess.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
