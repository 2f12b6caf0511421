// lz_ops.cu — Codec::lz per-op entry points of the C ABI on the device:
// lz_encode / lz_decode (codec.hpp:223-244) over host buffers, one warp per
// chunk (lz.cuh).  Encoding runs the parse twice: lengths first (a host
// prefix sum places the chunks), then the payload bytes at their offsets —
// byte-identical to the reference (tests/test_gpu_lz_codec.py).
#include <cstring>
#include <vector>

#include "common.cuh"
#include "lz.cuh"

namespace wg {
namespace {

// One warp per chunk; T: table entry type (16-bit when every chunk fits).
template <typename T>
__global__ void __launch_bounds__(32) k_lz_encode(const unsigned char* in, uint64_t n, uint64_t chunk,
                                                  const uint64_t* out_off, unsigned char* out, uint64_t* enc_len) {
    extern __shared__ __align__(16) unsigned char lz_smem[];
    T* table = reinterpret_cast<T*>(lz_smem);
    const uint64_t c = blockIdx.x;
    const uint64_t off = c * chunk;
    const uint32_t len = (uint32_t)(n - off < chunk ? n - off : chunk);
    const uint32_t m = lz_chunk_warp<T>(in + off, len, table, out ? out + out_off[c] : nullptr);
    if (!out && threadIdx.x == 0) enc_len[c] = m;
}

__global__ void __launch_bounds__(32) k_lz_decode(const unsigned char* in, const uint64_t* in_off,
                                                  const uint64_t* enc_len, uint64_t n, uint64_t chunk,
                                                  unsigned char* out, int* err) {
    const uint64_t c = blockIdx.x;
    const uint64_t off = c * chunk;
    const uint32_t raw = (uint32_t)(n - off < chunk ? n - off : chunk);
    const int e = lz_decode_chunk_warp(in + in_off[c], (uint32_t)enc_len[c], raw, out + off);
    if (threadIdx.x == 0) err[c] = e;
}

}  // namespace

// lz_encode of a device buffer (n bytes + >= 16 B of tail padding) in chunks
// of `chunk` bytes: the per-chunk payload lengths and the payloads back to
// back, on the host (session checkpoints, wg_lz_encode).
void lz_encode_device(const unsigned char* d_in, uint64_t n, uint64_t chunk, std::vector<uint64_t>& len,
                      std::vector<unsigned char>* payload) {
    const uint64_t nc = (n + chunk - 1) / chunk;
    len.assign(nc, 0);
    if (payload) payload->clear();
    if (nc == 0) return;
    if (nc > 0x7FFFFFFFull || chunk > 0xFFFFFFFFull) raise(WG_INVALID_ARGUMENT, "lz_encode: sizes out of range");
    DevBuf<uint64_t> d_len(nc);
    const bool small = chunk <= 65535;
    const size_t smem = small ? 8192 * sizeof(uint16_t) : 8192 * sizeof(uint32_t);
    auto launch = [&](const uint64_t* off, unsigned char* dst) {
        if (small) k_lz_encode<uint16_t><<<(unsigned)nc, 32, smem>>>(d_in, n, chunk, off, dst, d_len.p);
        else k_lz_encode<uint32_t><<<(unsigned)nc, 32, smem>>>(d_in, n, chunk, off, dst, d_len.p);
        WG_LAUNCH_CHECK("lz encode");
        WG_CUDA(cudaDeviceSynchronize());
    };
    launch(nullptr, nullptr);  // payload lengths
    d_len.download(len.data());
    if (!payload) return;
    std::vector<uint64_t> off(nc);
    uint64_t tot = 0;
    for (uint64_t c = 0; c < nc; ++c) {
        off[c] = tot;
        tot += len[c];
    }
    DevBuf<uint64_t> d_off(nc);
    d_off.upload(off.data());
    DevBuf<unsigned char> d_out(tot + 1);
    launch(d_off.p, d_out.p);  // the payload bytes
    payload->resize(tot);
    if (tot) WG_CUDA(cudaMemcpy(payload->data(), d_out.p, tot, cudaMemcpyDeviceToHost));
}

}  // namespace wg

using namespace wg;

extern "C" {

wg_status wg_lz_encode(const uint8_t* data, uint64_t n, uint64_t chunk, uint8_t* out, uint64_t cap,
                       uint64_t* enc_len, uint64_t* out_len) {
    return guard([&] {
        if (chunk == 0) raise(WG_INVALID_ARGUMENT, "lz_encode: chunk_size must be > 0");
        if (out_len) *out_len = 0;
        if (n == 0) return;
        DevBuf<unsigned char> d_in(n + 16);  // tail padding for the 8-byte word loads
        WG_CUDA(cudaMemcpy(d_in.p, data, n, cudaMemcpyHostToDevice));
        WG_CUDA(cudaMemset(d_in.p + n, 0, 16));
        std::vector<uint64_t> len;
        std::vector<unsigned char> pl;
        lz_encode_device(d_in.p, n, chunk, len, out ? &pl : nullptr);
        uint64_t tot = 0;
        for (size_t c = 0; c < len.size(); ++c) {
            if (enc_len) enc_len[c] = len[c];
            tot += len[c];
        }
        if (out_len) *out_len = tot;
        if (!out) return;
        if (tot > cap) raise(WG_OUT_OF_RANGE, "lz_encode: output buffer too small");
        std::memcpy(out, pl.data(), tot);
    });
}

wg_status wg_lz_decode(const uint8_t* payload, const uint64_t* enc_len, uint64_t chunk, uint8_t* out, uint64_t n) {
    return guard([&] {
        if (chunk == 0) raise(WG_INVALID_ARGUMENT, "lz_decode: chunk_size must be > 0");
        const uint64_t nc = (n + chunk - 1) / chunk;
        if (nc == 0) return;
        if (chunk > 0xFFFFFFFFull || nc > 0x7FFFFFFFull) raise(WG_INVALID_ARGUMENT, "lz_decode: sizes out of range");
        std::vector<uint64_t> off(nc);
        uint64_t tot = 0;
        for (uint64_t c = 0; c < nc; ++c) {
            if (enc_len[c] > 0xFFFFFFFFull) raise(WG_CORRUPT_STREAM, "lz_decode: truncated chunk");
            off[c] = tot;
            tot += enc_len[c];
        }
        DevBuf<unsigned char> d_in(tot + 16), d_out(n);
        if (tot) WG_CUDA(cudaMemcpy(d_in.p, payload, tot, cudaMemcpyHostToDevice));
        DevBuf<uint64_t> d_off(nc), d_len(nc);
        d_off.upload(off.data());
        d_len.upload(enc_len);
        DevBuf<int> d_err(nc);
        k_lz_decode<<<(unsigned)nc, 32>>>(d_in.p, d_off.p, d_len.p, n, chunk, d_out.p, d_err.p);
        WG_LAUNCH_CHECK("lz decode");
        WG_CUDA(cudaDeviceSynchronize());
        std::vector<int> err(nc);
        d_err.download(err.data());
        static const char* why[] = {"", "lz_decode: truncated chunk", "lz_decode: raw_len overrun",
                                    "lz_decode: bad match offset", "lz_decode: trailing bytes"};
        for (uint64_t c = 0; c < nc; ++c)  // the first corrupt chunk in stream order (lz_decode's throw)
            if (err[c]) raise(WG_CORRUPT_STREAM, why[err[c]]);
        d_out.download(out);
    });
}

}  // extern "C"
