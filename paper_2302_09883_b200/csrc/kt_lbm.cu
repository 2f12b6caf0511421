// kt_lbm.cu — D2Q9 step kernels (persistent, 3 rounds x 3 populations) and
// the opt-in half-line variant.
#include <cstdlib>
#include <string>

#include "half_kernels.cuh"
#include "kt_common.cuh"
#include "lbm_kernels.cuh"

namespace wg {
namespace {

template <int N, int L>
struct FullL {
    static KernelSet make() {
        using Lay = LbmLayout<N>;
        return KernelSet{k_lbm_step<N, L, MODE_STEP>, k_lbm_step<N, L, MODE_DECODE>, k_lbm_step<N, L, MODE_INIT>,
                         1, Lay::NT, Lay::smem_bytes(), true, Lay::scratch_doubles(), true, false,
                         k_lbm_step<N, L, MODE_STEP_LZ>};
    }
};

template <int N, int L>
struct HalfL {
    static KernelSet make() {
        using Lay = HLayout<N, 3>;
        return KernelSet{k_lbm_step_h<N, L, MODE_STEP>, k_lbm_step_h<N, L, MODE_DECODE>, nullptr, 1, Lay::NT,
                         Lay::smem_bytes(), true, LbmLayout<N>::scratch_doubles(), false, false};
    }
};

}  // namespace

bool select_lbm_kernels(uint64_t n, int levels, bool half_lines, KernelSet& k) {
    switch (n) {
        case 17: return pick_level<FullL, 17, 6>(levels, k);
        case 33: return pick_level<FullL, 33, 6>(levels, k);
        case 65: {
            const char* lines = std::getenv("WG_LBM_LINES");  // "group": 8-lane line groups
            if (lines && std::string(lines) == "group") return select_lbm_group_kernels(levels, k);
            return half_lines ? pick_level<HalfL, 65, 6>(levels, k) : pick_level<FullL, 65, 6>(levels, k);
        }
        default: return false;
    }
}

}  // namespace wg
