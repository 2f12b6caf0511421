// kt_transport.cu — transport (1 component) step kernels: k_patch_step
// (P patches per CTA).
#include "kt_common.cuh"
#include "patch_kernels.cuh"

// patches per CTA, measured at 4096^2: 65-point patches 3 per CTA (7 warps
// at 1 CTA/SM: 97 GLUPS; 2 -> 74, 4 -> 67), 33-point patches 7 per CTA
// (256 threads at 2 CTAs/SM: 113 GLUPS; 4 -> 91, 5 -> 105, 6 -> 103,
// 8 -> 87, 12 -> 63)
#ifndef WG_T65_P
#define WG_T65_P 3
#endif
#ifndef WG_T33_P
#define WG_T33_P 7
#endif

namespace wg {
namespace {

template <int P>
struct FullT {
    template <int N, int L>
    struct M {
        static KernelSet make() {
            using Lay = Layout<N, P>;
            return KernelSet{k_patch_step<N, L, P, MODE_STEP>, k_patch_step<N, L, P, MODE_DECODE>, nullptr, P,
                             Lay::NT, Lay::smem_bytes(), false, 0, false, true, k_patch_step<N, L, P, MODE_STEP_LZ>};
        }
    };
};

}  // namespace

bool select_transport_kernels(uint64_t n, int levels, bool small_grid, KernelSet& k) {
    if (small_grid && n == 33) return pick_level<FullT<1>::M, 33, kMaxLevels>(levels, k);
    switch (n) {
        case 9: return pick_level<FullT<7>::M, 9, kMaxLevels>(levels, k);
        case 17: return pick_level<FullT<15>::M, 17, kMaxLevels>(levels, k);
        case 33: return pick_level<FullT<WG_T33_P>::M, 33, kMaxLevels>(levels, k);
        case 65: return pick_level<FullT<WG_T65_P>::M, 65, kMaxLevels>(levels, k);
        default: return false;
    }
}

}  // namespace wg
