// kt_lbm17.cu — D2Q9 step kernels for 17-point patches (lbm_pair.cuh: one
// patch per 2-CTA cluster; step, Codec::lz step, decode and device initial
// state).  One translation unit per patch side / level range so the
// instantiations build in parallel.
#include "kt_lbm.cuh"

namespace wg {

bool select_lbm17(int levels, KernelSet& k) { return pick_level<PairL, 17, 4, 0>(levels, k); }

}  // namespace wg
