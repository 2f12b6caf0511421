// common.cuh — status handling shared by the C ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "wavegrid_b200.h"

namespace wg {

// C++ exception carrying a wg_status; converted at the ABI boundary.
struct Error : std::runtime_error {
    wg_status status;
    Error(wg_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void raise(wg_status s, const std::string& m) { throw Error(s, m); }

void set_last_error(const std::string& m);

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        raise(e == cudaErrorMemoryAllocation ? WG_OUT_OF_MEMORY : WG_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define WG_CUDA(call) ::wg::cuda_check((call), #call)
#define WG_LAUNCH_CHECK(what) ::wg::cuda_check(cudaGetLastError(), what)

// Run f and translate exceptions into a wg_status (no exception crosses the
// C ABI).
template <typename F>
wg_status guard(F&& f) {
    try {
        f();
        return WG_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return WG_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return WG_LOGIC;
    }
}

// Device buffer owned by a host scope (per-op entry points).
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) : n(count) {
        if (count) WG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void upload(const T* h) {
        if (n) WG_CUDA(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
    }
    void download(T* h) const {
        if (n) WG_CUDA(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost));
    }
};

// Device-side error word bits.
enum : unsigned {
    ERR_STORE_OVERFLOW = 1u << 0,
    ERR_CORRUPT = 1u << 1,
    ERR_DOMAIN = 1u << 2,
    ERR_RIEMANN = 1u << 3,
    ERR_RAW_OVERFLOW = 1u << 4,
    ERR_ZERO_SPEED = 1u << 5,
    ERR_PEER_TIMEOUT = 1u << 6,
    ERR_CONSISTENCY = 1u << 7,
};

inline void check_device_error(unsigned word) {
    if (!word) return;
    if (word & ERR_STORE_OVERFLOW)
        raise(WG_OUT_OF_MEMORY, "compressed patch store exceeded its budget");
    if (word & ERR_RAW_OVERFLOW) raise(WG_OUT_OF_MEMORY, "raw-patch list overflow");
    if (word & ERR_CORRUPT) raise(WG_CORRUPT_STREAM, "csr_decode: invalid block");
    if (word & ERR_DOMAIN) raise(WG_DOMAIN, "water depth must be positive");
    if (word & ERR_RIEMANN) raise(WG_RIEMANN, "SweRiemann: Newton iteration did not converge");
    if (word & ERR_ZERO_SPEED) raise(WG_INVALID_ARGUMENT, "cfl_dt: zero wave speed");
    if (word & ERR_CONSISTENCY) raise(WG_CONSISTENCY, "assemble: shared cells disagree");
    if (word & ERR_PEER_TIMEOUT) raise(WG_LOGIC, "peer halo exchange: a neighbour shard did not deliver its halo lines");
    raise(WG_LOGIC, "device error word " + std::to_string(word));
}

constexpr int kMaxRank = 8;

}  // namespace wg
