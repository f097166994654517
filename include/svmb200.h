/*
 * svmb200.h -- C ABI of the B200-native SMO SVM solver (libsvmb200.so).
 *
 * The library trains a binary soft-margin kernel SVM by SMO on NVIDIA B200 (sm_100a)
 * and evaluates batched decision values.  Sources of the operations:
 *   PAPER.md  = Elgarhy, "Support Vector Machine Implementation on MPI-CUDA and
 *               Tensorflow Framework" (arXiv 2311.14908), cited "P:L<line>"
 *   SPEC.md   = the derived CPU specification, cited "S:L<line>"
 *
 *   svm_train / svm_train_ex   the SMO solve of the dual QP
 *       max_a  sum a_i - 1/2 sum_ij a_i a_j y_i y_j K(x_i, x_j)
 *       s.t.   0 <= a_i <= C,  sum a_i y_i = 0                      (§3.1-3.2)
 *     two multipliers per step "under the KKT constraints", the maximal
 *     violating pair with lowest-index ties, f_i = sum_j a_j y_j K_ij - y_i, stop when
 *     b_low - b_up <= 2 tol, b = -(b_up + b_low)/2
 *     Kernels: linear x.z and RBF exp(-gamma ||x - z||^2)
 *   svm_predict                dec(x) = sum_s coef_s K(x_s, x) + b
 *   svm_train_gd_dev           the paper's gradient-descent (TensorFlow) trainer read as
 *                              projected gradient ascent on the same dual
 *
 * Row storage is chosen per solve and never changes the arithmetic: fp32 rows; bit rows
 * when every value is 0 or 1; mixed bit / fp32 rows when >= 32 columns are 0/1; one-byte
 * dictionary codes when X has <= 256 distinct values (svm_last_plan() reports which).
 *
 * Arithmetic contract: X is float32; every kernel value,
 * the error vector f, the multipliers and all reductions are fp64; distances and
 * dot products accumulate in ascending feature order with one fma per term; exp is
 * correctly rounded.  Results are therefore identical to any implementation of the
 * same readings (the repository's CPU oracle) bit for bit, and independent of the
 * number of GPUs / CTAs the rows are spread over.
 *
 * Conventions
 *   - Return value: SVM_OK (0) or a negative svm_status; svm_last_error() gives a
 *     thread-local message for the last failing call on the calling thread.
 *   - Non-convergence (max_iter reached) is success with info->converged = 0.
 *   - Host entry points take host pointers; the caller owns every buffer, the library
 *     copies inputs in and keeps no pointer after return.  Device entry points take
 *     device pointers on the caller's stream and allocate only scratch, freed before
 *     return.
 *   - Layout: X row-major [n][d] float32; y int8 in {+1,-1}; alpha, f, coef, dec fp64.
 *   - Calls are not re-entrant on one communicator.
 */
#ifndef SVMB200_H
#define SVMB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { SVM_LINEAR = 0, SVM_RBF = 1 } svm_kernel;

typedef enum {
    SVM_OK = 0,
    SVM_EINVAL = -1,        /* n < 2, d < 1, C <= 0 or non-finite, tol <= 0, RBF gamma <= 0, null pointer */
    SVM_ELABEL = -2,        /* a label outside {+1, -1} */
    SVM_ESINGLECLASS = -3,  /* all labels equal */
    SVM_ENONFINITE = -4,    /* NaN / Inf in X */
    SVM_ENOMEM = -5,        /* device allocation failed, or a shard too large for the SMEM-resident state */
    SVM_ECUDA = -6,         /* CUDA runtime error (message in svm_last_error) */
    SVM_ENCCL = -7,         /* NCCL error during communicator setup */
    SVM_ETIMEOUT = -8       /* a device-side wait for another CTA / rank exceeded its watchdog */
} svm_status;

/* Solver controls.  Zero / negative fields take the defaults shown. */
typedef struct {
    double C;               /* box bound, > 0 */
    double gamma;           /* RBF width, > 0 (ignored for linear) */
    double tol;             /* tau; <= 0 -> 1e-3; converged when b_low - b_up <= 2 tau */
    int64_t max_iter;       /* <= 0 -> max(10 n, 10000) */
    int32_t check_interval; /* <= 0 -> 64: the host-visible progress word is refreshed every
                               check_interval iterations ("convergence checks ... for every set
                               of iterations"); results do not depend on it */
    int32_t kernel;         /* svm_kernel */
    double sv_epsilon;      /* <= 0 -> 1e-8: support set {alpha > sv_epsilon} */
    int32_t virtual_ranks;  /* <= 1 -> 1.  >1 splits the rows of ONE GPU into that many ranks
                               that run the full multi-rank exchange protocol among CTA groups
                               (test hook for the row-sharded path; results are identical) */
    int32_t ctas;           /* <= 0 -> one CTA per SM; else the CTA count (test hook) */
    int64_t iters_per_launch; /* <= 0 -> unlimited: the whole solve is one persistent launch */
    int32_t gram;           /* full-Gram path: 1 force (one rank), otherwise off.
                               K is precomputed once with the same arithmetic (R13/R14), so
                               results are identical either way. */
    int32_t cache_rows;     /* kernel-row cache: > 0 slots, -1 off, 0 auto (X
                               streamed from HBM and n <= 200,000: max(64, n/25) slots, at most
                               2048).  A slot holds the kernel row K(i, .) restricted to each CTA's
                               own rows; every CTA runs the same directory (hash lookup, FIFO
                               replacement) on the same pair sequence.  An iteration whose two
                               rows are both cached reads them (and K_ul) instead of streaming X.
                               Cached values are the computed ones, so results are identical. */
    int32_t cluster;        /* candidate exchange among a rank's CTAs: 0 auto, -1 global-memory
                               mailboxes, 1..16 force one thread-block cluster of that many CTAs
                               per rank exchanging through distributed shared memory (one rank
                               or batched problems; the rank's rows must fit resident in the
                               cluster's shared memory).  Auto picks a cluster when the rows fit
                               (<= 2048 rows per CTA, or <= 8192 with 16 CTAs).  The exchange
                               computes the same lexicographic winner, so results are identical. */
    int32_t wss;            /* working-set selection: <= 1 the maximal violating pair (DESIGN
                               reading R1); 2 second order (Fan, Chen & Lin 2005, cited at P:L140):
                               u as in 1, then l = argmax over t in I_low with f_t > f_u of
                               (f_t - f_u)^2 / (K_uu + K_tt - 2 K_ut), lowest index on ties; the
                               stopping test stays b_low - b_up <= 2 tol.  Each iteration then
                               takes two row passes and two exchanges.  Not for
                               svm_train_batch_dev. */
    int32_t shrink_window;  /* window shrinking (DESIGN reading R29): 0 off; H > 0 runs the solve in
                               windows of H updates; at each window start (every row selected
                               over, stopping test taken) the rows that cannot form a violating
                               pair -- i in I_up only with f_i > b_low, i in I_low only with
                               f_i < b_up -- are set aside for the window: only the active rows
                               are streamed and selected over, and the window's updates are
                               replayed on the rows set aside at its end (their f stays the exact
                               incremental value).  A window also ends when the active rows'
                               gap reaches 2 tol.  svm_train_dev / svm_train_ex, one rank. */
    int32_t reserved1;      /* 0 */
} svm_params;

typedef struct {
    int64_t iterations;     /* SMO pair updates performed */
    int32_t converged;      /* 1: b_low - b_up <= 2 tol;  0: stopped at max_iter */
    int32_t n_sv;           /* |{alpha > sv_epsilon}| */
    double gap;             /* final b_low - b_up */
    double b_up, b_low;     /* final min f over I_up, max f over I_low */
    double dual_objective;  /* W = 1/2 sum_i alpha_i (1 - y_i f_i) */
    double seconds_solve;   /* device time of the solver launches (CUDA events) */
    double seconds_total;   /* host wall time of the call, including H2D / D2H */
    int64_t launches;       /* persistent-kernel launches used */
    int64_t cache_hits;     /* kernel-row cache (a8): row lookups served from the cache (two per
                               SMO iteration: x_up's row and x_low's row) */
    int64_t cache_misses;   /* row lookups that computed the row (and filled a slot) */
    double seconds_h2d;     /* host entry points: device time of the H2D copy of X and y (0 for
                               device entry points) */
} svm_info;

/* Optional debug / test hooks; a NULL svm_debug costs nothing.  Host entry points
 * (svm_train_ex) take host pointers for alpha0 / f0 / f_out; device entry points
 * (svm_train_dev, svm_train_shard) take DEVICE pointers for them, of the rank's rows
 * ([n_local], the rank's slice) for svm_train_shard.  pair_trace is always a host pointer
 * (svm_train_shard: filled on rank 0 only).  A warm start resumes a saved state: the
 * solve continues from (alpha0, f0) exactly as the interrupted solve would have
 * (segment parity). */
typedef struct {
    const double* alpha0;     /* warm start [n] (both alpha0 and f0, or neither) */
    const double* f0;         /* warm start [n]: the error vector matching alpha0 */
    double* f_out;            /* [n] out: final f */
    int64_t* pair_trace;      /* [2 * pair_trace_cap] out: (i_up, i_low) of each update */
    int64_t pair_trace_cap;
} svm_debug;

/* Train on host data.  alpha: [n] out (dense, zeros for non-SVs); b: out. */
int svm_train(const float* X, const int8_t* y, int64_t n, int64_t d, double C, int kernel,
              double gamma, double tol, double* alpha, double* b);

/* Train on host data with full controls; info and dbg may be NULL. */
int svm_train_ex(const float* X, const int8_t* y, int64_t n, int64_t d, const svm_params* p,
                 double* alpha, double* b, svm_info* info, const svm_debug* dbg);

/* Train on device data already resident in HBM (X row-major [n][d] float32, y int8),
 * on `cuda_stream` (cudaStream_t, NULL = legacy default).  alpha (device, [n]) out,
 * b and info host out (n_sv and the dual objective are reduced on the device); dbg:
 * alpha0 / f0 / f_out device pointers, pair_trace host. */
int svm_train_dev(const float* X, const int8_t* y, int64_t n, int64_t d, const svm_params* p,
                  double* alpha, double* b, svm_info* info, const svm_debug* dbg,
                  void* cuda_stream);

/* B independent binary problems with the same controls, solved concurrently: one
 * persistent launch splits the SMs into up to 8 CTA groups, each running its own SMO loop
 * and exchange (no communication between problems; more than 8 problems run in successive
 * launches).  This is the within-GPU form of the paper's task-parallel multiclass training
 * ("running multiple parallel binary SMOs", Fig. 4).  Device pointers: X[k]
 * row-major [n[k]][d] float32, y[k] int8, alpha[k] [n[k]] out; b_out[B] and info[B]
 * (nullable) host out.  Each result equals svm_train_dev on that problem alone. */
int svm_train_batch_dev(int B, const float* const* X, const int8_t* const* y, const int64_t* n,
                        int64_t d, const svm_params* p, double* const* alpha, double* b_out,
                        svm_info* info, void* cuda_stream);

/* Decision values of m test rows (host pointers): dec[i] = sum_s coef_s K(sv_s, x_i) + b
 * with coef_s = alpha_s y_s, summed in ascending s in fp64.  n_sv = 0 gives
 * dec = b. */
int svm_predict(const float* X_sv, const double* coef, int64_t n_sv, int64_t d, double b,
                int kernel, double gamma, const float* X_test, int64_t m, double* dec);

/* Same on device pointers and the caller's stream. */
int svm_predict_dev(const float* X_sv, const double* coef, int64_t n_sv, int64_t d, double b,
                    int kernel, double gamma, const float* X_test, int64_t m, double* dec,
                    void* cuda_stream);

/* Prediction mode.  EXACT: fp64 SIMT, the arithmetic of R13/R14/R19, decision
 * values bit-identical to any implementation of those readings.  TENSOR: the contraction
 * T * SV^T on the 5th-generation tensor cores (tcgen05.mma kind::tf32, operands split
 * "3xTF32" = hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM) with an fp64 epilogue
 * (distance, exp, coefficient sum); BASELINE.json tolerance 1e-4 absolute. */
typedef enum { SVM_PREDICT_EXACT = 0, SVM_PREDICT_TENSOR = 1 } svm_predict_mode;

int svm_predict_ex(const float* X_sv, const double* coef, int64_t n_sv, int64_t d, double b,
                   int kernel, double gamma, const float* X_test, int64_t m, double* dec,
                   int mode);
int svm_predict_dev_ex(const float* X_sv, const double* coef, int64_t n_sv, int64_t d, double b,
                       int kernel, double gamma, const float* X_test, int64_t m, double* dec,
                       int mode, void* cuda_stream);

/* The support set of a trained model, compacted on the device (row a10):
 * {i : alpha_i > sv_epsilon} (sv_epsilon <= 0 -> 1e-8) in ascending i.  Device pointers:
 * X [n][d] float32, y int8, alpha [n] fp64 in; X_sv [n_sv][d] float32, coef [n_sv] fp64
 * (coef_i = alpha_i y_i, exact), sv_index [n_sv] int64 out (sv_index nullable; X_sv
 * nullable).  With coef == NULL only *n_sv (host) is written, so a caller can size the
 * outputs first; otherwise the outputs must hold n_sv entries.  Synchronises the stream. */
int svm_support_vectors_dev(const float* X, const int8_t* y, const double* alpha, int64_t n,
                            int64_t d, double sv_epsilon, float* X_sv, double* coef,
                            int64_t* sv_index, int64_t* n_sv, void* cuda_stream);

/* ---- multi-GPU, one process per GPU (torchrun) -----------------------------------
 * svm_comm_unique_id fills 128 bytes on rank 0 that the caller broadcasts (e.g. with
 * torch.distributed); every rank then calls svm_comm_init (NCCL bootstrap).  Or every rank
 * calls svm_comm_init_host with a host all-gather callback (any transport, e.g. gloo;
 * also the only option for several ranks on ONE device, which NCCL refuses).
 * svm_train_shard trains on the rank's contiguous row block [row_offset, row_offset +
 * n_local) of an n_global-row problem; every rank must call it with the same parameters.
 * Device pointers; alpha_local receives the rank's slice of alpha.  Each iteration, every
 * CTA stores its 64-byte candidate record into every rank's mailbox (peer stores through
 * CUDA IPC mappings over NVLink); a record is four 16-byte words whose two 8-byte halves
 * each carry the exchange's sequence number, so a reader accepts only whole words
 * (8-byte accesses are single-copy atomic).  Results are bit-identical for any number of
 * ranks.  dbg: alpha0 / f0 / f_out device pointers of the rank's rows, pair_trace host
 * (rank 0). */
typedef struct {
    void* ctx;
    /* every rank passes `bytes` bytes in send; recv (host, world * bytes) receives every
     * rank's bytes in rank order.  Returns 0 on success. */
    int (*allgather)(void* ctx, const void* send, void* recv, int64_t bytes);
} svm_host_coll;

int svm_comm_unique_id(uint8_t id[128]);
int svm_comm_init(void** comm, int rank, int world, const uint8_t id[128], int device);
int svm_comm_init_host(void** comm, int rank, int world, int device, const svm_host_coll* coll);
int svm_train_shard(void* comm, const float* X_local, const int8_t* y_local, int64_t n_local,
                    int64_t row_offset, int64_t n_global, int64_t d, const svm_params* p,
                    double* alpha_local, double* b, svm_info* info, const svm_debug* dbg,
                    void* cuda_stream);
void svm_comm_destroy(void* comm);

/* ---- projected-gradient dual trainer ------------------------
 * The paper's TensorFlow path (§3.3, Fig. 5: "declaring the gradient descent
 * optimizer algorithm") read as full-batch projected gradient ascent on the same dual W
 * (R23-R26): from alpha = 0, `epochs` times
 *     g = K (alpha o y)   (g_i summed in ascending j, one fma per term),
 *     alpha_i <- min(C, max(0, fma(lr, 1 - y_i g_i, alpha_i))),
 * then b = mean of y_i - g_i over 1e-8 < alpha_i < C - 1e-8 (else -(max g + min g)/2 over
 * the alpha_i > 1e-8, else over all i) and W = sum alpha - 1/2 sum alpha_i y_i g_i for the
 * final alpha.  The equality constraint sum alpha y = 0 is not enforced (box projection
 * only).  K is the full fp64 kernel matrix (R13/R14/R16), built once in HBM (8 n^2 bytes;
 * SVM_ENOMEM when it does not fit); every epoch streams it once.
 * Device pointers X [n][d] float32 row-major, y int8 (+1/-1), alpha [n] out; b, info host
 * out (info nullable).  lr > 0 finite, epochs >= 0.  Errors as svm_train_dev. */
typedef struct {
    double objective;        /* W(alpha) of the returned alpha */
    double seconds_gram;     /* device time of building K */
    double seconds_epochs;   /* device time of the epochs (+ the final evaluation pass) */
    int64_t epochs;
    int64_t gram_bytes;      /* bytes of K in HBM (column blocks of one CTA each, zero padded) */
} svm_gd_info;

int svm_train_gd_dev(const float* X, const int8_t* y, int64_t n, int64_t d, double C, int kernel,
                     double gamma, double lr, int64_t epochs, double* alpha, double* b,
                     svm_gd_info* info, void* cuda_stream);

/* Number of CUDA kernels this library has launched from the calling thread so far
 * (validation, staging, the persistent solver launches, prediction). */
int64_t svm_kernel_launches(void);

/* How the last solve on this thread ran (observability, not part of the arithmetic): a
 * one-line JSON object, e.g. {"kernel": "smo_bincl<1>", "ctas_per_rank": 16, "cluster": 16,
 * "mode": "binary-resident", "threads": 256, "smem": 73488}.  "" before the first solve. */
const char* svm_last_plan(void);

/* Message for the last non-OK status returned on this thread ("" if none). */
const char* svm_last_error(void);

/* Library version string, e.g. "svmb200 0.1 sm_100a". */
const char* svm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SVMB200_H */
