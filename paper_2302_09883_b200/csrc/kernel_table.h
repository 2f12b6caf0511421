// kernel_table.h — the fused step kernels of a session, chosen at session
// creation from (scheme, patch side, levels).  Every instantiation lives in
// one translation unit per scheme (kt_*.cu) so the builds run in parallel.
#pragma once

#include <cstddef>
#include <cstdint>

namespace wg {

struct StepArgs;

struct KernelSet {
    void (*main)(StepArgs);
    void (*decode)(StepArgs);
    void (*init)(StepArgs);  // device-generated, compressed initial state (D2Q9); may be null
    int P;                   // patches per CTA (non-persistent kernels)
    int threads;
    size_t smem;
    bool persistent;         // grid-stride over patches with per-CTA scratch
    size_t scratch_doubles;  // per CTA
    bool edges3;             // D2Q9 edge lines hold only the 3 crossing populations
    bool decode_l2;          // decode with decode_out == nullptr runs the transport l2 pass
    void (*main_lz)(StepArgs) = nullptr;  // MODE_STEP_LZ (Codec::lz metrics); null if unsupported
    int cluster = 1;                      // CTAs per patch (thread-block cluster size of every mode)
};

// Each returns false when (n, levels) has no instantiation.
// small_grid: fewer patches than the CTAs of a full wave at the default
// patches-per-CTA: one patch per CTA spreads them over more SMs
bool select_transport_kernels(uint64_t n, int levels, bool small_grid, KernelSet& out);  // kt_transport.cu
bool select_lbm_kernels(uint64_t n, int levels, KernelSet& out);        // kt_lbm.cu
bool select_swe_kernels(uint64_t n, int levels, KernelSet& out);                         // kt_swe*.cu
bool select_swe65_kernels(int levels, KernelSet& out);                                  // kt_swe65.cu

// Raises WG_INVALID_ARGUMENT when unsupported (session.cu).
KernelSet select_kernels(int scheme, uint64_t n, int levels, uint64_t npatch);

}  // namespace wg
