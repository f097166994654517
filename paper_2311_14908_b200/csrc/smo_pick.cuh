// smo_pick.cuh -- the solver kernel's instantiations, chosen at run time by svmb200.cu's
// pick_kernel.  Included only by the four smo_{gen,spec}_{rbf,lin}.cu translation units, so
// the ~110 instantiations of smo_persistent compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "smo_kernel.cuh"

namespace svmint {

using svmk::NT;
using svmk::Params;
using svmk::smo_persistent;

typedef void (*KernelFn)(const Params);

// SPEC 1-3 (mixed / dense / dictionary rows only); nullptr when no specialisation applies
template <int K, bool W>
KernelFn pick_spec_w(int rpt, bool a_smem, int ntc, bool mix, bool dense, bool dict) {
    if (ntc == NT && dict && !W && rpt >= 2) {
        if (a_smem) return rpt == 4 ? smo_persistent<K, 4, true, false, NT, false, false, 3> : smo_persistent<K, 2, true, false, NT, false, false, 3>;
        return rpt == 4 ? smo_persistent<K, 4, false, false, NT, false, false, 3> : smo_persistent<K, 2, false, false, NT, false, false, 3>;
    }
    if (ntc == NT && dense && rpt >= 2) {
        if (a_smem) return rpt == 4 ? smo_persistent<K, 4, true, false, NT, false, W, 2> : smo_persistent<K, 2, true, false, NT, false, W, 2>;
        return rpt == 4 ? smo_persistent<K, 4, false, false, NT, false, W, 2> : smo_persistent<K, 2, false, false, NT, false, W, 2>;
    }
    if (ntc == 448 && mix) {
        if (a_smem) return rpt == 2 ? smo_persistent<K, 2, true, false, 448, false, W, 1> : smo_persistent<K, 1, true, false, 448, false, W, 1>;
        return rpt == 2 ? smo_persistent<K, 2, false, false, 448, false, W, 1> : smo_persistent<K, 1, false, false, 448, false, W, 1>;
    }
    if (ntc == 512 && mix) {
        if (a_smem) return rpt == 2 ? smo_persistent<K, 2, true, false, 512, false, W, 1> : smo_persistent<K, 1, true, false, 512, false, W, 1>;
        return rpt == 2 ? smo_persistent<K, 2, false, false, 512, false, W, 1> : smo_persistent<K, 1, false, false, 512, false, W, 1>;
    }
    return nullptr;
}

template <int K>
KernelFn pick_spec_k(int rpt, bool a_smem, int ntc, bool wide, bool mix, bool dense, bool dict) {
    return wide ? pick_spec_w<K, true>(rpt, a_smem, ntc, mix, dense, false)
                : pick_spec_w<K, false>(rpt, a_smem, ntc, mix, dense, dict);
}

// SPEC 0: every mode compiled in (16 warps: no binary rows / row cache)
template <int K, bool W>
KernelFn pick_general_w(int rpt, bool a_smem, int ntc) {
    if (ntc == 512) {
        if (a_smem) return rpt == 2 ? smo_persistent<K, 2, true, false, 512, false, W> : smo_persistent<K, 1, true, false, 512, false, W>;
        return rpt == 2 ? smo_persistent<K, 2, false, false, 512, false, W> : smo_persistent<K, 1, false, false, 512, false, W>;
    }
    if (a_smem) return rpt == 4 ? smo_persistent<K, 4, true, false, NT, false, W> : rpt == 2 ? smo_persistent<K, 2, true, false, NT, false, W> : smo_persistent<K, 1, true, false, NT, false, W>;
    return rpt == 4 ? smo_persistent<K, 4, false, false, NT, false, W> : rpt == 2 ? smo_persistent<K, 2, false, false, NT, false, W> : smo_persistent<K, 1, false, false, NT, false, W>;
}

// wss2: the second-order selection (256 consumers); wide: the consumer-warp record poll
template <int K>
KernelFn pick_general_k(int rpt, bool a_smem, int ntc, bool wss2, bool wide) {
    if (wss2) {
        if (a_smem) return rpt == 4 ? smo_persistent<K, 4, true, false, NT, true> : rpt == 2 ? smo_persistent<K, 2, true, false, NT, true> : smo_persistent<K, 1, true, false, NT, true>;
        return rpt == 4 ? smo_persistent<K, 4, false, false, NT, true> : rpt == 2 ? smo_persistent<K, 2, false, false, NT, true> : smo_persistent<K, 1, false, false, NT, true>;
    }
    return wide ? pick_general_w<K, true>(rpt, a_smem, ntc) : pick_general_w<K, false>(rpt, a_smem, ntc);
}

// binary rows resident in a cluster (BINCL: every other mode compiled out)
template <int K>
KernelFn pick_bincl_spec_k(bool a_smem) {
    return a_smem ? smo_persistent<K, 1, true, true> : smo_persistent<K, 1, false, true>;
}

}  // namespace svmint
