// smo_spec_lin.cu -- the specialised instantiations (mixed / dense / dictionary rows only, binary rows in a cluster) of
// smo_persistent for the linear kernel (smo_pick.cuh); one translation unit of four so they
// compile in parallel.
#include "smo_pick.cuh"

namespace svmint {

KernelFn pick_spec_lin(int rpt, bool a_smem, int ntc, bool wide, bool mix, bool dense, bool dict) {
    return pick_spec_k<0>(rpt, a_smem, ntc, wide, mix, dense, dict);
}
KernelFn pick_bincl_spec_lin(bool a_smem) { return pick_bincl_spec_k<0>(a_smem); }

}  // namespace svmint
