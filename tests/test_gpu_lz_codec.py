"""Codec::lz bytes on the device (csrc/lz.cuh, csrc/lz_ops.cu): the product's
lz_encode / lz_decode — one warp per chunk — against the reference compiled
unchanged (oracle/_ref), byte for byte (codec.hpp:127-244), including the
real thresholded coefficient arrays of a D2Q9 step and the corrupt-stream
checks of lz_decode_chunk."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api

from .lz_cases import CHUNKS, corruptions, lz_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chunk", CHUNKS)
def test_lz_encode_decode_bytes(product, reference, chunk):
    for name, data in lz_inputs(big=chunk >= 65535).items():
        if chunk < 64 and len(data) > 70000:
            continue
        got = api.lz_encode(data, chunk, lib=product)
        want = api.lz_encode(data, chunk, lib=reference)
        assert got[1] == want[1], (name, "payload lengths")
        assert got[0] == want[0], (name, "payload bytes")
        assert api.lz_decode(want[0], want[1], chunk, len(data), lib=product) == data, name


def test_lz_thresholded_coefficients(product, reference, oracle):
    """The arrays the Codec::lz run compresses: apply_threshold's output of
    every population block of a C2-shaped D2Q9 patch (-0.0 kept)."""
    cfg = api.RunConfig(scheme="lbm", nx=129, splits=(2, 2), levels=4, lbm_steps=3,
                        spec=api.ThresholdSpec("capped", 1e-3))
    g = api.run(cfg, lib=oracle).grid
    for p in range(4):
        for q in range(9):
            blk = np.ascontiguousarray(g.data[p, q, 1:-1, 1:-1])
            cs = api.dwt_nd(blk, 4, lib=oracle)
            api.apply_threshold(cs, 4, cfg.spec, lib=oracle)
            data = np.ascontiguousarray(cs).tobytes()
            assert api.lz_encode(data, 64 * 1024, lib=product) == api.lz_encode(data, 64 * 1024, lib=reference)


def test_lz_decode_rejects_corrupt_streams(product, reference):
    data = lz_inputs()["smooth_f64"][:4000]
    pl, lens = api.lz_encode(data, 1 << 16, lib=reference)
    for name, p2, l2 in corruptions(pl, lens):
        with pytest.raises(abi.CorruptStreamError):
            api.lz_decode(p2, l2, 1 << 16, len(data), lib=product)
    with pytest.raises(abi.InvalidArgument):
        api.lz_encode(b"abc", 0, lib=product)
