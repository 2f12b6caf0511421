// kt_lbm.cuh — the D2Q9 KernelSet (lbm_pair.cuh) shared by the kt_lbm*.cu units.
#pragma once

#include "kt_common.cuh"
#include "lbm_pair.cuh"

namespace wg {

template <int N, int L>
struct PairL {
    static KernelSet make() {
        using Lay = PairLayout<N>;
        KernelSet k{k_lbm_pair<N, L, MODE_STEP>, k_lbm_pair<N, L, MODE_DECODE>, k_lbm_pair<N, L, MODE_INIT>,
                    1, Lay::NT, Lay::smem_bytes(), true, 0, true, false, k_lbm_pair<N, L, MODE_STEP_LZ>};
        k.cluster = 2;
        return k;
    }
};

bool select_lbm17(int levels, KernelSet& k);
bool select_lbm33(int levels, KernelSet& k);
bool select_lbm65a(int levels, KernelSet& k);
bool select_lbm65b(int levels, KernelSet& k);
bool select_lbm65c(int levels, KernelSet& k);

}  // namespace wg
