// smo_spec_rbf.cu -- the specialised instantiations (mixed / dense / dictionary rows only, binary rows in a cluster) of
// smo_persistent for the RBF kernel (smo_pick.cuh); one translation unit of four so they
// compile in parallel.
#include "smo_pick.cuh"

namespace svmint {

KernelFn pick_spec_rbf(int rpt, bool a_smem, int ntc, bool wide, bool mix, bool dense, bool dict) {
    return pick_spec_k<1>(rpt, a_smem, ntc, wide, mix, dense, dict);
}
KernelFn pick_bincl_spec_rbf(bool a_smem) { return pick_bincl_spec_k<1>(a_smem); }

}  // namespace svmint
