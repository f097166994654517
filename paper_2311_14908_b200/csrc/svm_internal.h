// svm_internal.h -- shared declarations of the host driver (not part of the ABI).
#pragma once
#include <vector>

#include <cuda_runtime.h>

#include <string>

#include "../../include/svmb200.h"
#include "smo_kernel.cuh"

namespace svmint {

extern thread_local std::string g_err;
extern thread_local std::string g_plan;            // svm_last_plan
int fail(int code, const std::string& msg);
// kernels this library launched from the calling thread (svm_kernel_launches)
extern thread_local long long g_launches;
inline void counted(long long k = 1) { g_launches += k; }

#define CKR(x)                                                                          \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess)                                                          \
            return ::svmint::fail(SVM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct SolveOut {
    long long iterations = 0;
    int state = 0;
    double b_up = 0, b_low = 0;
    double seconds_solve = 0;
    long long launches = 0;
    long long cache_hits = 0, cache_misses = 0;
    bool gram = false;
    bool plain_rows = false;                   // the solve streamed plain fp32 rows (no encoding)
};

struct SolveArgs;
typedef int (*PreLaunchFn)(SolveArgs&, svmk::Params&);

struct SolveArgs {
    svm_params p;
    long long n_global = 0, d = 0;
    const float* xr = nullptr;                 // row-major replica [n_global][d] (device)
    int world = 1, rank_base = 0, nranks_here = 1, ctas_per_rank = 1;
    int n_sm = 0, max_smem = 0;
    long long n_rows_max = 0;
    long long row_off[svmk::MAXR] = {};
    long long n_rows[svmk::MAXR] = {};
    const float* x_rank[svmk::MAXR] = {};      // device rows of rank r, row-major
    const int8_t* y_rank[svmk::MAXR] = {};
    double* alpha_out[svmk::MAXR] = {};        // device alpha of rank r's rows
    svmk::Mailbox* mbox[svmk::MAXR] = {};      // all ranks (peer pointers) unless local alloc
    bool mbox_local_alloc = true;
    const double* alpha0 = nullptr;            // device warm start: global indexing if warm_global,
    const double* f0 = nullptr;                //   else the served rank's rows
    bool warm_global = true;
    double* f_out = nullptr;                   // destination of f (global indexing if f_out_global)
    cudaMemcpyKind f_out_kind = cudaMemcpyDeviceToHost;
    bool f_out_global = true;
    long long* trace = nullptr;                // host
    long long trace_cap = 0;
    long long* trace_dev = nullptr;            // device pair trace + (c_u, c_l) history, written
    double* hist_dev = nullptr;                //   by the kernel in place (window shrinking)
    long long dev_cap = 0;
    bool skip_detect = false;                  // plain fp32 rows without probing X for encodings
    cudaStream_t stream = nullptr;
    long long timeout_ns = 20ll * 1000 * 1000 * 1000;
    PreLaunchFn pre_launch = nullptr;
    void* user = nullptr;
    bool independent = false;                  // batched independent problems (one per rank)
    const float* xr_rank[svmk::MAXR] = {};
    long long max_iter_rank[svmk::MAXR] = {};
    std::vector<int> mix_map;                  // (set by solve) mixed compact rows: column map
    std::vector<double> dict_vals;             // (set by solve) dictionary-coded rows: values,
    std::vector<unsigned> dict_keys;           //   the value set (fp32 bit patterns, hashed)
    std::vector<unsigned char> dict_code;      //   and the code of every set slot
    SolveOut out;                              // rank_base's result
    SolveOut out_rank[svmk::MAXR];             // every served rank (independent mode)
};

int check_params(long long n, long long d, const svm_params* p, svm_params* q);
int validate_device(const float* X, const int8_t* y, long long n, long long d, cudaStream_t st,
                    int* n_pos);
int device_limits(int* n_sm, int* max_smem);
void pool_setup();
int solve(SolveArgs& a);
int train_device(const float* X, const int8_t* y, long long n, long long d, const svm_params& p,
                 double* alpha, const double* alpha0, const double* f0, double* f_out,
                 cudaMemcpyKind f_kind, long long* trace, long long trace_cap, cudaStream_t st,
                 SolveOut& out, long long* trace_dev = nullptr, double* hist_dev = nullptr,
                 long long dev_cap = 0, bool skip_detect = false);
// shrink.cu: window shrinking (R29) around train_device, one rank
int train_shrink(const float* X, const int8_t* y, long long n, long long d, const svm_params& p,
                 double* alpha, const double* alpha0, const double* f0, double* f_out,
                 long long* trace, long long trace_cap, cudaStream_t st, SolveOut& out);

// gram.cu: K[i][j] for all i, j < n (fp64, row-major), same arithmetic as the row pass
int gram_device(const float* X, long long n, long long d, int kernel, double gamma, double* K,
                cudaStream_t st, long long ld = 0, int blk = 0);

// finalize.cu: out_host = {sum alpha_i (1 - y_i f_i), n_sv} over n rows (device pointers)
int info_device(const double* alpha, const double* f, const int8_t* y, long long n, double eps,
                cudaStream_t st, double out_host[2]);

// predict.cu
int predict_device(const float* X_sv, const double* coef, long long n_sv, long long d, double b,
                   int kernel, double gamma, const float* X_test, long long m, double* dec,
                   cudaStream_t st, int mode);

}  // namespace svmint
