// kt_lbm.cu — D2Q9 kernel selection by patch side and level count (the
// instantiations live in kt_lbm17/33/65{a,b,c}.cu).
#include "kernel_table.h"
#include "kt_lbm.cuh"

namespace wg {

bool select_lbm_kernels(uint64_t n, int levels, KernelSet& k) {
    switch (n) {
        case 17: return select_lbm17(levels, k);
        case 33: return select_lbm33(levels, k);
        case 65: return levels <= 3 ? select_lbm65a(levels, k) : levels == 4 ? select_lbm65b(levels, k)
                                                                               : select_lbm65c(levels, k);
        default: return false;
    }
}

}  // namespace wg
