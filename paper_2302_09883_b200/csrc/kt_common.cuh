// kt_common.cuh — KernelSet construction shared by the kt_*.cu units.
#pragma once

#include "common.cuh"
#include "kernel_table.h"
#include "patch_phases.cuh"

namespace wg {

inline void kt_set_smem(const KernelSet& k) {
    int dev = 0, optin = 0;
    WG_CUDA(cudaGetDevice(&dev));
    WG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    for (auto f : {k.main, k.decode, k.init, k.main_lz})
        if (f) {
            cudaFuncAttributes fa{};
            WG_CUDA(cudaFuncGetAttributes(&fa, f));
            if (fa.sharedSizeBytes + k.smem > (size_t)optin)
                raise(WG_LOGIC, "kernel shared memory (static " + std::to_string(fa.sharedSizeBytes) + " + dynamic " +
                                    std::to_string(k.smem) + ") exceeds the per-block limit");
            WG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem));
        }
}

// Walk L = 0.. while 2^L <= N-1 (and L <= Lmax); Make<N, L>::make() builds the set.
template <template <int, int> class Make, int N, int Lmax, int L = 0>
bool pick_level(int levels, KernelSet& out) {
    static_assert(L >= 0);
    if constexpr ((1 << L) <= N - 1 && L <= Lmax) {
        if (levels == L) {
            out = Make<N, L>::make();
            kt_set_smem(out);
            return true;
        }
        return pick_level<Make, N, Lmax, L + 1>(levels, out);
    } else {
        return false;
    }
}

}  // namespace wg
