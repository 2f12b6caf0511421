// lz.cuh — Codec::lz on the device (codec.hpp:81-244): the reference's greedy
// LZ77 parse of one chunk by ONE WARP, producing the exact payload length and,
// when an output pointer is given, the payload bytes themselves — byte for
// byte what lz_encode_chunk (codec.hpp:127-175) emits; and the warp decoder
// of a chunk (lz_decode_chunk, codec.hpp:177-220) with its corruption checks.
//
// Parse (reference semantics, restated): a 13-bit hash of the 4 bytes at the
// current position selects a table slot holding the last position with that
// hash; the slot is overwritten by the current position; a candidate within
// 65535 bytes whose first 4 bytes match starts a match, extended to the first
// differing byte (or the chunk end); the sequence (literals since the anchor,
// match) is emitted and the parse resumes after the match (positions inside a
// match are never inserted).  Output of a sequence: a token (literal count in
// the high nibble, match length - 4 in the low one, 15 = "extended by 255-byte
// runs"), the literal-length extension, the literals, the 2-byte
// little-endian offset, the match-length extension; the chunk ends with a
// literal-only sequence (token low nibble 0) when literals remain.
//
// Warp mapping: 32 candidate positions are probed per step (each lane sees
// the table exactly as the sequential parse would: the latest lower lane with
// the same hash, else the table — __match_any_sync), the lowest lane with a
// match ends the window, only the positions up to it are inserted (latest
// per hash); matches are extended 256-1024 bytes per round by ballots; the
// literals of a sequence are copied by all 32 lanes.
#pragma once

#include <cstdint>

namespace wg {

// Unaligned 8-byte little-endian load (the input has >= 8 B of tail padding
// or the caller stays 8 B inside it).
__device__ __forceinline__ uint64_t lz_load8(const unsigned char* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~uintptr_t(7));
    const unsigned sh = (unsigned)(a & 7) * 8;
    const uint64_t lo = w[0];
    return sh ? (lo >> sh) | (w[1] << (64 - sh)) : lo;
}

// Bytes of a length extension (lz_put_length, codec.hpp:113-119).
__device__ __forceinline__ uint32_t lz_ext_bytes(uint32_t len) { return len / 255 + 1; }

// Writes the extension of `len` at out[o] (lane 0); returns the new o.
__device__ __forceinline__ uint32_t lz_put_ext(unsigned char* out, uint32_t o, uint32_t len, int lane) {
    const uint32_t nb = lz_ext_bytes(len);
    for (uint32_t k = lane; k < nb; k += 32) out[o + k] = k + 1 < nb ? (unsigned char)255 : (unsigned char)(len - 255 * (nb - 1));
    return o + nb;
}

// One sequence at out[o]: token, literal extension, the literals in[anchor,
// anchor + lit), then (ml >= 0) the offset and the match extension.
// Returns the new o.  All lanes call it (the literal copy is warp-wide).
__device__ __forceinline__ uint32_t lz_put_sequence(unsigned char* out, uint32_t o, const unsigned char* in,
                                                    uint32_t anchor, uint32_t lit, int ml, uint32_t offset,
                                                    int lane) {
    const uint32_t ln = lit < 15 ? lit : 15;
    const uint32_t mn = ml < 0 ? 0u : ((uint32_t)ml < 15 ? (uint32_t)ml : 15u);
    if (lane == 0) out[o] = (unsigned char)((ln << 4) | mn);
    ++o;
    if (ln == 15) o = lz_put_ext(out, o, lit - 15, lane);
    for (uint32_t k = lane; k < lit; k += 32) out[o + k] = in[anchor + k];
    o += lit;
    if (ml < 0) return o;
    if (lane == 0) {
        out[o] = (unsigned char)(offset & 0xff);
        out[o + 1] = (unsigned char)(offset >> 8);
    }
    o += 2;
    if (mn == 15) o = lz_put_ext(out, o, (uint32_t)ml - 15, lane);
    return o;
}

// The parse of one chunk in[0, n) by a whole warp with a per-warp hash table
// of 8192 entries (T: uint16_t when n <= 65535, else uint32_t; the maximum
// value marks an empty slot).  Returns the payload length; writes the payload
// to out when out != nullptr.
template <typename T>
__device__ uint32_t lz_chunk_warp(const unsigned char* in, uint32_t n, T* table, unsigned char* out) {
    const int lane = threadIdx.x & 31;
    constexpr T kEmpty = (T)~T(0);
    for (int k = lane; k < 8192; k += 32) table[k] = kEmpty;
    __syncwarp();
    uint32_t anchor = 0, pos = 0, o = 0;
    auto ext = [](uint32_t len) { return len / 255 + 1; };
    while (n >= 4 && pos + 4 <= n) {
        const uint32_t w = pos + lane;
        const bool act = w + 4 <= n;
        const uint32_t v = act ? (uint32_t)lz_load8(in + w) : 0u;
        const uint32_t h = (v * 2654435761u) >> 19;
        const unsigned actm = __ballot_sync(0xffffffffu, act);
        const unsigned peers = __match_any_sync(0xffffffffu, act ? h : 0xFFFFFFFFu) & actm;
        const unsigned lower = peers & ((1u << lane) - 1u);
        const T tv = act && !lower ? table[h] : kEmpty;
        const long long cand = !act ? -1 : lower ? (long long)(pos + 31 - __clz(lower)) : (tv == kEmpty ? -1 : (long long)tv);
        const bool hit = act && cand >= 0 && w - (uint32_t)cand <= 65535u && (uint32_t)lz_load8(in + cand) == v;
        const unsigned hits = __ballot_sync(0xffffffffu, hit);
        const int first = hits ? __ffs(hits) - 1 : 31;
        const unsigned upto = (first == 31) ? actm : (actm & ((2u << first) - 1u));
        // insert the processed positions: per hash the latest one wins
        const unsigned later = peers & upto & ~((2u << lane) - 1u);
        __syncwarp();
        if (((upto >> lane) & 1u) && !later) table[h] = (T)w;
        __syncwarp();
        if (!hits) {
            pos += __popc(actm);  // all literals
            continue;
        }
        const uint32_t mpos = pos + first;
        const uint32_t mc = (uint32_t)__shfl_sync(0xffffffffu, (long long)cand, first);
        uint32_t len = 4;
        for (;;) {
            if (mpos + len + 1024 <= n) {  // 1 KiB per round: 4 independent word pairs per lane in flight
                uint64_t d[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    d[u] = lz_load8(in + mc + len + 256 * u + 8 * lane) ^ lz_load8(in + mpos + len + 256 * u + 8 * lane);
                bool stop = false;
#pragma unroll
                for (int u = 0; u < 4 && !stop; ++u) {
                    const unsigned m = __ballot_sync(0xffffffffu, d[u] != 0);
                    if (!m) {
                        len += 256;
                        continue;
                    }
                    const int f = __ffs(m) - 1;
                    const uint64_t df = __shfl_sync(0xffffffffu, d[u], f);
                    len += 8 * f + (uint32_t)(__ffsll((long long)df) - 1) / 8;
                    stop = true;
                }
                if (stop) break;
                continue;
            }
            if (mpos + len + 256 <= n) {
                const uint64_t d = lz_load8(in + mc + len + 8 * lane) ^ lz_load8(in + mpos + len + 8 * lane);
                const unsigned m = __ballot_sync(0xffffffffu, d != 0);
                if (!m) {
                    len += 256;
                    continue;
                }
                const int f = __ffs(m) - 1;
                const uint64_t df = __shfl_sync(0xffffffffu, d, f);
                len += 8 * f + (uint32_t)(__ffsll((long long)df) - 1) / 8;
                break;
            }
            while (mpos + len < n && in[mc + len] == in[mpos + len]) ++len;  // the tail (< 256 B)
            break;
        }
        const uint32_t lit = mpos - anchor, ml = len - 4;
        if (out) o = lz_put_sequence(out, o, in, anchor, lit, (int)ml, mpos - mc, lane);
        else o += 1 + (lit >= 15 ? ext(lit - 15) : 0) + lit + 2 + (ml >= 15 ? ext(ml - 15) : 0);
        pos = mpos + len;
        anchor = pos;
    }
    if (anchor < n) {  // the terminal literal-only sequence
        const uint32_t lit = n - anchor;
        if (out) o = lz_put_sequence(out, o, in, anchor, lit, -1, 0, lane);
        else o += 1 + (lit >= 15 ? ext(lit - 15) : 0) + lit;
    }
    __syncwarp();
    return o;
}

// lz_decode_chunk (codec.hpp:177-220) by a warp: the token stream is parsed
// in lock-step by every lane, literal runs and matches copied lane-parallel
// (a match whose offset is shorter than 32 bytes copies offset bytes per
// round: the overlap semantics of the byte loop).  Returns 0 or a reason:
// 1 truncated chunk, 2 raw_len overrun, 3 bad match offset, 4 trailing bytes.
__device__ inline int lz_decode_chunk_warp(const unsigned char* in, uint32_t in_len, uint32_t raw_len,
                                           unsigned char* out) {
    const int lane = threadIdx.x & 31;
    uint32_t p = 0, o = 0;
    auto get_length = [&](uint32_t base, int& err) -> uint32_t {
        uint32_t len = base;
        if (base == 15) {
            unsigned b;
            do {
                if (p + 1 > in_len) {
                    err = 1;
                    return 0;
                }
                b = in[p++];
                len += b;
            } while (b == 255);
        }
        return len;
    };
    while (o < raw_len) {
        if (p + 1 > in_len) return 1;
        const unsigned token = in[p++];
        int err = 0;
        const uint32_t lit = get_length(token >> 4, err);
        if (err) return err;
        if (p + lit > in_len) return 1;
        if (o + lit > raw_len) return 2;
        for (uint32_t k = lane; k < lit; k += 32) out[o + k] = in[p + k];
        p += lit;
        o += lit;
        __syncwarp();
        if (o == raw_len) break;
        if (p + 2 > in_len) return 1;
        const uint32_t offset = (uint32_t)in[p] | ((uint32_t)in[p + 1] << 8);
        p += 2;
        const uint32_t ml = get_length(token & 0x0f, err) + 4;
        if (err) return err;
        if (offset == 0 || offset > o) return 3;
        if (o + ml > raw_len) return 2;
        const uint32_t step = offset < 32 ? offset : 32;
        for (uint32_t base = 0; base < ml; base += step) {
            const uint32_t k = base + lane;
            unsigned char c = 0;
            if (lane < (int)step && k < ml) c = out[o - offset + k];
            __syncwarp();
            if (lane < (int)step && k < ml) out[o + k] = c;
            __syncwarp();
        }
        o += ml;
    }
    return p != in_len ? 4 : 0;
}

}  // namespace wg
