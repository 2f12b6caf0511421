// kt_swe65.cu — shallow-water step kernels for 65-point patches.
#include "kt_common.cuh"
#include "swe_kernels.cuh"

namespace wg {

template <int N, int L>
struct SweK65 {
    static KernelSet make() {
        using Lay = SweLayout<N>;
        return KernelSet{k_swe_step<N, L, MODE_STEP>, k_swe_step<N, L, MODE_DECODE>, nullptr, 1, Lay::NT,
                         Lay::smem_bytes(), true, Lay::scratch_doubles(), false, false,
                         k_swe_step<N, L, MODE_STEP_LZ>};
    }
};

bool select_swe65_kernels(int levels, KernelSet& k) { return pick_level<SweK65, 65, 6>(levels, k); }

}  // namespace wg
