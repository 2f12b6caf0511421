"""Shared Codec::lz inputs (codec.hpp:81-244) for the CPU and GPU codec
tests: random, compressible, adversarial (long runs, repeats at offsets
around the 65535 window and the hash-table size, tiny chunks) and real
thresholded coefficient arrays; plus corrupt-stream mutations."""
from __future__ import annotations

import numpy as np


def lz_inputs(big: bool = False):
    rng = np.random.default_rng(2302)
    n = 1 << (20 if big else 16)
    cases = {
        "empty": b"",
        "short": b"abc",
        "zeros": bytes(n),
        "random": rng.integers(0, 256, n, dtype=np.uint8).tobytes(),
        "period8": (b"abcdefgh" * (n // 8 + 1))[: n + 3],
        "smooth_f64": np.sin(np.arange(n // 8) * 0.001).tobytes(),
        "sparse_f64": np.where(rng.random(n // 8) < 0.05, rng.standard_normal(n // 8), 0.0).tobytes(),
        "few_symbols": rng.integers(0, 3, n, dtype=np.uint8).tobytes(),
    }
    # a block repeated at distances 65535, 65536 and 70000: the offset limit
    blk = rng.integers(0, 256, 300, dtype=np.uint8).tobytes()
    far = bytearray(rng.integers(0, 256, 140300, dtype=np.uint8).tobytes())
    for at in (0, 65535, 65535 + 65536, 140000):
        far[at: at + 300] = blk
    cases["far_repeats"] = bytes(far)
    # runs longer than 255 / 270 bytes (length extensions) between literals
    cases["runs"] = b"".join(bytes([k % 7]) * (k * 37 % 700 + 1) + bytes([k % 256, 255 - k % 256]) for k in range(300))
    return cases


CHUNKS = (7, 64, 4096, 65535, 65536, 1 << 20)


def corruptions(payload: bytes, enc_len: list):
    """(name, payload, enc_len) mutations of a one-chunk stream that
    lz_decode_chunk rejects."""
    out = []
    if enc_len and enc_len[0] > 2:
        out.append(("truncated", payload[:-1], [enc_len[0] - 1] + enc_len[1:]))
        out.append(("trailing", payload[: enc_len[0]] + b"\x00" + payload[enc_len[0]:], [enc_len[0] + 1] + enc_len[1:]))
    return out
