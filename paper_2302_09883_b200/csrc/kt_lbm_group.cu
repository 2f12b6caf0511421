// kt_lbm_group.cu — D2Q9 step kernels with 8-lane line groups
// (lbm_group_kernels.cuh), 65-point patches.
#include "kt_common.cuh"
#include "lbm_group_kernels.cuh"

namespace wg {

template <int N, int L>
struct GroupL {
    static KernelSet make() {
        using Lay = GLayout<N>;
        return KernelSet{k_lbm_step_g<N, L, MODE_STEP>, k_lbm_step_g<N, L, MODE_DECODE>,
                         k_lbm_step_g<N, L, MODE_INIT>, 1, Lay::NT, Lay::smem_bytes(), true,
                         Lay::scratch_doubles(), true, false};
    }
};

bool select_lbm_group_kernels(int levels, KernelSet& k) { return pick_level<GroupL, 65, 6>(levels, k); }

}  // namespace wg
