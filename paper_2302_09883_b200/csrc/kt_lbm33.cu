// kt_lbm33.cu — D2Q9 step kernels for 33-point patches (lbm_pair.cuh: one
// patch per 2-CTA cluster; step, Codec::lz step, decode and device initial
// state).  One translation unit per patch side / level range so the
// instantiations build in parallel.
#include "kt_lbm.cuh"

namespace wg {

bool select_lbm33(int levels, KernelSet& k) { return pick_level<PairL, 33, 5, 0>(levels, k); }

}  // namespace wg
