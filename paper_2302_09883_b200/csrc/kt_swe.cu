// kt_swe.cu — shallow-water step kernels for patch sides 9, 17, 33
// (65: kt_swe65.cu, a separate unit so the two compile in parallel).
#include "kt_common.cuh"
#include "swe_kernels.cuh"

namespace wg {

template <int N, int L>
struct SweK {
    static KernelSet make() {
        using Lay = SweLayout<N>;
        return KernelSet{k_swe_step<N, L, MODE_STEP>, k_swe_step<N, L, MODE_DECODE>, nullptr, 1, Lay::NT,
                         Lay::smem_bytes(), true, Lay::scratch_doubles(), false, false,
                         k_swe_step<N, L, MODE_STEP_LZ>};
    }
};

bool select_swe_kernels(uint64_t n, int levels, KernelSet& k) {
    switch (n) {
        case 9: return pick_level<SweK, 9, 6>(levels, k);
        case 17: return pick_level<SweK, 17, 6>(levels, k);
        case 33: return pick_level<SweK, 33, 6>(levels, k);
        case 65: return select_swe65_kernels(levels, k);
        default: return false;
    }
}

}  // namespace wg
