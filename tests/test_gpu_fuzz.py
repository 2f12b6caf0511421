"""Seeded random configurations of the fused loop against the C oracle (all
three schemes, every supported patch side, levels up to the patch depth,
every threshold mode, shards, tiny and uneven grids): the broad net behind
the hand-picked parity cases."""
from __future__ import annotations

import random

import pytest

from paper_2302_09883_b200 import api

from .test_gpu_session import compare_runs

pytestmark = pytest.mark.gpu

SIDES = {"transport": (9, 17, 33, 65), "swe": (9, 17, 33, 65), "lbm": (17, 33, 65)}


def _cases(n=90, seed=2302):
    rng = random.Random(seed)
    out = []
    for k in range(n):
        scheme = ("transport", "swe", "lbm")[k % 3]
        side = rng.choice(SIDES[scheme])
        depth = (side - 1).bit_length() - 1
        splits = rng.choice((1, 2, 3, 4)) if side <= 33 else rng.choice((1, 2))
        nx = (side - 1) * splits + 1
        levels = rng.randint(0, depth)
        mode = rng.choice(("constant", "accumulation", "capped"))
        c = rng.choice((0.0, 1e-5, 1e-4, 1e-3, 1e-2, 5e-2))
        out.append((scheme, nx, splits, levels, mode, c, rng.randint(1, 6)))
    return out


@pytest.mark.parametrize("scheme,nx,splits,levels,mode,c,steps", _cases())
def test_random_config(product, oracle_sq, scheme, nx, splits, levels, mode, c, steps):
    spec = api.ThresholdSpec(mode, c)
    if scheme == "lbm":
        cfg = api.RunConfig(scheme="lbm", nx=nx, splits=(splits, splits), levels=levels, lbm_steps=steps, spec=spec)
    else:
        cfg = api.RunConfig(scheme=scheme, nx=nx, splits=(splits, splits), levels=levels, spec=spec,
                            compute_l2=False)
        dx = 1.0 / (nx - 1)
        cfg.t_end = steps * cfg.cfl * dx / (0.9 if scheme == "transport" else 4.5)
    compare_runs(api.run(cfg, lib=product), api.run(cfg, lib=oracle_sq))
