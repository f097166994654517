// Host build of the CUDA path's exp (paper_2311_14908_b200/csrc/svm_exp.cuh) for
// CPU tests of its correct rounding.  Test helper only.
#include "../../paper_2311_14908_b200/csrc/svm_exp.cuh"
extern "C" double svm_exp_host(double x) { return svmexp::exp_cr(x); }
extern "C" long svm_exp_host_batch(const double* x, double* out, long n) {
    for (long i = 0; i < n; ++i) out[i] = svmexp::exp_cr(x[i]);
    return n;
}
