"""Checkpoint / resume straight from the device's compressed store
(wg_session_save / wg_session_load).

A session saved after k steps and resumed in a fresh session continues bit
for bit like the uninterrupted one; every WGC1 record of the file decodes
(with the reference's container and codec semantics, api.load_wgc /
decode_patch, and the C oracle's idwt) to the session's state at the save."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2302_09883_b200 import abi, api

from .test_gpu_session import bits

pytestmark = pytest.mark.gpu


def _cfg(scheme):
    if scheme == "transport":
        cfg = api.RunConfig(scheme="transport", nx=129, splits=(4, 4), levels=4, t_end=1.0,
                            spec=api.ThresholdSpec("capped", 1e-3))
    elif scheme == "lbm":
        cfg = api.RunConfig(scheme="lbm", nx=129, splits=(2, 2), levels=4, lbm_steps=100,
                            spec=api.ThresholdSpec("capped", 1e-3))
    else:
        cfg = api.RunConfig(scheme="swe", nx=129, splits=(4, 4), levels=4, t_end=1.0,
                            spec=api.ThresholdSpec("constant", 5e-4))
    return cfg


class _S:
    def __init__(self, lib, cfg):
        self.lib, self.cfg = lib, cfg
        c = cfg.to_c()
        self.h = abi.vp()
        lib.check(lib.wg_session_create(C.byref(c), None, None, C.byref(self.h)))
        self.info = abi.SessionInfoC()
        lib.check(lib.wg_session_info_get(self.h, C.byref(self.info)))

    def close(self):
        self.lib.wg_session_destroy(self.h)

    def steps(self, k):
        dt = self.cfg.cfl / (self.cfg.nx - 1) / 0.9
        for _ in range(k):
            self.lib.check(self.lib.wg_session_step(self.h, dt))

    def state(self):
        n = self.info.npatch_local * self.info.components * (self.info.patch_n + 2) ** 2
        out = np.zeros(n)
        self.lib.check(self.lib.wg_session_download(self.h, abi.dptr(out)))
        return out

    def rows(self):
        n = abi.u64()
        self.lib.check(self.lib.wg_session_metrics(self.h, None, 0, C.byref(n)))
        buf = (abi.MetricsRowC * max(n.value, 1))()
        self.lib.check(self.lib.wg_session_metrics(self.h, buf, n.value, C.byref(n)))
        return [(r.step, r.time, r.nnz, r.zeroed, r.compressed_bytes) for r in buf[: n.value]]


@pytest.mark.parametrize("scheme", ["transport", "lbm", "swe"])
def test_resume_is_bit_identical(product, oracle, tmp_path, scheme):
    cfg = _cfg(scheme)
    g0 = api.initial_state(cfg, lib=product)
    ck = tmp_path / "state.wgs"
    a = _S(product, cfg)
    b = _S(product, cfg)
    try:
        product.check(product.wg_session_upload(a.h, abi.dptr(g0.data)))
        a.steps(4)
        product.check(product.wg_session_save(a.h, str(ck).encode()))
        at_save = a.state()
        a.steps(5)
        final_a, rows_a = a.state(), a.rows()[4:]
        product.check(product.wg_session_load(b.h, str(ck).encode()))
        assert np.array_equal(bits(b.state()), bits(at_save))
        b.steps(5)
        assert np.array_equal(bits(b.state()), bits(final_a))
        assert b.rows() == rows_a

        # the file: WGS1 header + one WGC1 record per patch, decodable with
        # the reference's container/codec semantics
        hdr, recs = api.read_checkpoint(ck)
        assert hdr["step"] == 4 and len(recs) == a.info.npatch_local
        n, m = a.info.patch_n, a.info.components
        view = at_save.reshape(len(recs), m, n + 2, n + 2)[:, :, 1:n + 1, 1:n + 1]
        kinds = set()
        for p, r in enumerate(recs):
            kinds.add(r.codec)
            coeffs = api.decode_patch(r, lib=oracle)
            for q in range(m):
                x = coeffs[q].reshape(n, n)
                field = api.idwt_nd(x, r.levels, lib=oracle) if r.levels else x
                assert np.array_equal(bits(field), bits(view[p, q])), (p, q, r.codec)
        assert 1 in kinds  # compressed records present
    finally:
        a.close()
        b.close()


def test_raw_patches_round_trip(product, reference, tmp_path):
    """c = 0: every patch is stored raw (skip rule) -> Codec::lz records whose
    payloads are the reference's own lz_encode of the block bytes (the device
    encoder, csrc/lz.cuh); -0.0 and every other bit pattern survive."""
    cfg = _cfg("swe")
    cfg.spec = api.ThresholdSpec("constant", 0.0)
    g0 = api.initial_state(cfg, lib=product)
    ck = tmp_path / "raw.wgs"
    a, b = _S(product, cfg), _S(product, cfg)
    try:
        product.check(product.wg_session_upload(a.h, abi.dptr(g0.data)))
        a.steps(3)
        product.check(product.wg_session_save(a.h, str(ck).encode()))
        _, recs = api.read_checkpoint(ck)
        assert {r.codec for r in recs} == {2} and all(r.levels == 0 for r in recs)
        state = a.state()
        n = recs[0].dims[0]
        tc = (n + 2) ** 2
        for p in (0, 5, len(recs) - 1):
            for q in range(recs[p].components):
                blk = state[(p * recs[p].components + q) * tc: (p * recs[p].components + q + 1) * tc].reshape(n + 2, n + 2)
                raw = np.ascontiguousarray(blk[1:-1, 1:-1]).tobytes()
                payload, lens = api.lz_encode(raw, 64 * 1024, lib=reference)
                chunk, chunks = recs[p].lz[q]
                assert chunk == 64 * 1024 and [c[0] for c in chunks] == [len(raw)]
                assert [len(c[1]) for c in chunks] == lens and chunks[0][1] == payload, (p, q)
        product.check(product.wg_session_load(b.h, str(ck).encode()))
        assert np.array_equal(bits(b.state()), bits(a.state()))
        a.steps(2)
        b.steps(2)
        assert np.array_equal(bits(b.state()), bits(a.state()))
    finally:
        a.close()
        b.close()


def test_load_rejects_foreign_and_corrupt_files(product, tmp_path):
    cfg = _cfg("transport")
    g0 = api.initial_state(cfg, lib=product)
    ck = tmp_path / "t.wgs"
    a = _S(product, cfg)
    other = api.RunConfig(scheme="transport", nx=129, splits=(2, 2), levels=4, t_end=1.0,
                          spec=api.ThresholdSpec("capped", 1e-3))
    b = _S(product, other)
    try:
        product.check(product.wg_session_upload(a.h, abi.dptr(g0.data)))
        a.steps(2)
        product.check(product.wg_session_save(a.h, str(ck).encode()))
        assert product.wg_session_load(b.h, str(ck).encode()) == 1  # WG_INVALID_ARGUMENT
        raw = bytearray(ck.read_bytes())
        raw[120:124] = b"XGC1"  # first record's magic
        bad = tmp_path / "bad.wgs"
        bad.write_bytes(bytes(raw))
        assert product.wg_session_load(a.h, str(bad).encode()) == 2  # WG_CORRUPT_STREAM
        trunc = tmp_path / "trunc.wgs"
        trunc.write_bytes(ck.read_bytes()[:-7])
        assert product.wg_session_load(a.h, str(trunc).encode()) == 2
    finally:
        a.close()
        b.close()
