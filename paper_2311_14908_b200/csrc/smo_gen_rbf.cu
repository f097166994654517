// smo_gen_rbf.cu -- the general instantiations (every mode, the second-order rule, the wide poll) of
// smo_persistent for the RBF kernel (smo_pick.cuh); one translation unit of four so they
// compile in parallel.
#include "smo_pick.cuh"

namespace svmint {

KernelFn pick_general_rbf(int rpt, bool a_smem, int ntc, bool wss2, bool wide) {
    return pick_general_k<1>(rpt, a_smem, ntc, wss2, wide);
}

}  // namespace svmint
