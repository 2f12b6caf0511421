// kt_lbm65c.cu — D2Q9 step kernels for 65-point patches, levels 5-6 (L = 6 = k: valid, not conservative) (lbm_pair.cuh: one
// patch per 2-CTA cluster; step, Codec::lz step, decode and device initial
// state).  One translation unit per patch side / level range so the
// instantiations build in parallel.
#include "kt_lbm.cuh"

namespace wg {

bool select_lbm65c(int levels, KernelSet& k) { return pick_level<PairL, 65, 6, 5>(levels, k); }

}  // namespace wg
