// comm.cu -- one process per GPU: communicator, peer mailboxes, svm_train_shard.
//
// The per-iteration exchange is device-initiated inside the
// persistent kernel: every CTA stores its 64-byte candidate record into every rank's
// mailbox through peer pointers (CUDA IPC mappings; NVLink when the ranks are GPUs) with
// system-scope relaxed stores; readers accept a 16-byte word only when both of its
// 8-byte halves carry the exchange's sequence number (smo_kernel.cuh).  The bootstrap --
// agreeing on the CTA count, exchanging the IPC handles, the one-time row-major replica
// of X used to gather the two pivot rows, a barrier before the first record, and the
// final n_sv / dual-objective sums -- runs over NCCL (svm_comm_init) or over a caller's
// host all-gather (svm_comm_init_host: any transport, and the only option for several
// ranks on one device, which NCCL refuses).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "svm_internal.h"

using namespace svmk;

namespace svmint {

struct Comm {
    ncclComm_t nccl = nullptr;
    svm_host_coll coll = {nullptr, nullptr};     // host bootstrap when nccl == nullptr
    int rank = 0, world = 1, device = 0;
    int ctas_per_rank = 0;
    int n_sm = 0, max_smem = 0;
    Mailbox* mbox_local = nullptr;
    size_t mbox_bytes = 0;
    Mailbox* peers[MAXR] = {};
    cudaStream_t st = nullptr;
};

#define CKN(x)                                                                          \
    do {                                                                                \
        ncclResult_t r_ = (x);                                                          \
        if (r_ != ncclSuccess)                                                          \
            return ::svmint::fail(SVM_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

// All-gather of `bytes` host bytes per rank into recv[world * bytes] (rank order).
int allgather_host(Comm* c, const void* send, void* recv, size_t bytes, cudaStream_t st) {
    if (!c->nccl) {
        if (c->coll.allgather(c->coll.ctx, send, recv, (int64_t)bytes) != 0)
            return fail(SVM_ENCCL, "host all-gather callback failed");
        return SVM_OK;
    }
    char* d;
    CKR(cudaMallocAsync(&d, bytes * c->world, st));
    CKR(cudaMemcpyAsync(d + bytes * c->rank, send, bytes, cudaMemcpyHostToDevice, st));
    CKN(ncclAllGather(d + bytes * c->rank, d, bytes, ncclChar, c->nccl, st));
    CKR(cudaMemcpyAsync(recv, d, bytes * c->world, cudaMemcpyDeviceToHost, st));
    CKR(cudaFreeAsync(d, st));
    CKR(cudaStreamSynchronize(st));
    return SVM_OK;
}

int comm_setup(Comm* c) {
    CKR(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    int rc = device_limits(&c->n_sm, &c->max_smem);
    if (rc) return rc;
    // agree on the CTA count per rank (minimum SM count over ranks)
    std::vector<int> sms(c->world);
    if ((rc = allgather_host(c, &c->n_sm, sms.data(), 4, c->st))) return rc;
    c->ctas_per_rank = sms[0];
    for (int r = 1; r < c->world; ++r) c->ctas_per_rank = sms[r] < c->ctas_per_rank ? sms[r] : c->ctas_per_rank;
    // mailbox + peer mapping
    c->mbox_bytes = svmk::mbox_bytes(c->ctas_per_rank, c->world);
    CKR(cudaMalloc(&c->mbox_local, c->mbox_bytes));
    CKR(cudaMemset(c->mbox_local, 0, c->mbox_bytes));
    cudaIpcMemHandle_t h;
    CKR(cudaIpcGetMemHandle(&h, c->mbox_local));
    std::vector<cudaIpcMemHandle_t> all(c->world);
    if ((rc = allgather_host(c, &h, all.data(), sizeof(h), c->st))) return rc;
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) { c->peers[r] = c->mbox_local; continue; }
        void* ptr = nullptr;
        CKR(cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess));
        c->peers[r] = (Mailbox*)ptr;
    }
    return SVM_OK;
}

void comm_free(Comm* c) {
    cudaSetDevice(c->device);
    for (int r = 0; r < c->world; ++r)
        if (r != c->rank && c->peers[r]) cudaIpcCloseMemHandle(c->peers[r]);
    if (c->mbox_local) cudaFree(c->mbox_local);
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

}  // namespace svmint

using namespace svmint;

extern "C" int svm_comm_unique_id(uint8_t id[128]) {
    if (!id) return fail(SVM_EINVAL, "null id");
    ncclUniqueId u;
    CKN(ncclGetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    memcpy(id, &u, 128);
    return SVM_OK;
}

extern "C" int svm_comm_init(void** out, int rank, int world, const uint8_t id[128], int device) {
    if (!out || !id) return fail(SVM_EINVAL, "null pointer");
    if (world < 1 || world > MAXR || rank < 0 || rank >= world)
        return fail(SVM_EINVAL, "world must be in [1, 8] and 0 <= rank < world");
    CKR(cudaSetDevice(device));
    Comm* c = new Comm;
    c->rank = rank; c->world = world; c->device = device;
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclResult_t nr = ncclCommInitRank(&c->nccl, world, u, rank);
    if (nr != ncclSuccess) { delete c; return fail(SVM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(nr)); }
    int rc = comm_setup(c);
    if (rc) { comm_free(c); return rc; }
    *out = c;
    return SVM_OK;
}

extern "C" int svm_comm_init_host(void** out, int rank, int world, int device, const svm_host_coll* coll) {
    if (!out || !coll || !coll->allgather) return fail(SVM_EINVAL, "null pointer");
    if (world < 1 || world > MAXR || rank < 0 || rank >= world)
        return fail(SVM_EINVAL, "world must be in [1, 8] and 0 <= rank < world");
    CKR(cudaSetDevice(device));
    Comm* c = new Comm;
    c->rank = rank; c->world = world; c->device = device;
    c->coll = *coll;
    int rc = comm_setup(c);
    if (rc) { comm_free(c); return rc; }
    *out = c;
    return SVM_OK;
}

extern "C" void svm_comm_destroy(void* comm) {
    Comm* c = (Comm*)comm;
    if (c) comm_free(c);
}

extern "C" int svm_train_shard(void* comm, const float* X_local, const int8_t* y_local,
                               int64_t n_local, int64_t row_offset, int64_t n_global, int64_t d,
                               const svm_params* p_in, double* alpha_local, double* b,
                               svm_info* info, const svm_debug* dbg, void* cuda_stream) {
    Comm* c = (Comm*)comm;
    if (!c || !X_local || !y_local || !alpha_local || !b) return fail(SVM_EINVAL, "null pointer");
    svm_params p;
    int rc = check_params(n_global, d, p_in, &p);
    if (rc) return rc;
    if (n_local < 0 || row_offset < 0 || row_offset + n_local > n_global)
        return fail(SVM_EINVAL, "row block outside [0, n_global)");
    if (dbg && ((dbg->alpha0 == nullptr) != (dbg->f0 == nullptr)))
        return fail(SVM_EINVAL, "warm start needs both alpha0 and f0");
    if (p.shrink_window > 0) return fail(SVM_EINVAL, "shrinking runs on one rank (svm_train_dev / svm_train_ex)");
    cudaStream_t st = cuda_stream ? (cudaStream_t)cuda_stream : c->st;
    CKR(cudaSetDevice(c->device));
    const int W = c->world;
    // ---- every rank's (row_offset, n_local)
    std::vector<long long> sz(2 * W);
    long long mine[2] = {row_offset, n_local};
    if ((rc = allgather_host(c, mine, sz.data(), 16, st))) return rc;
    long long covered = 0, n_max = 0;
    for (int r = 0; r < W; ++r) {
        if (sz[2 * r] != covered) return fail(SVM_EINVAL, "row blocks must be contiguous in rank order");
        covered += sz[2 * r + 1];
        n_max = sz[2 * r + 1] > n_max ? sz[2 * r + 1] : n_max;
    }
    if (covered != n_global) return fail(SVM_EINVAL, "row blocks do not cover n_global");
    // ---- the row-major replica of X (pivot rows are gathered from it) and y
    float* xr;
    int8_t* yr;
    CKR(cudaMallocAsync(&xr, (size_t)n_global * d * 4, st));
    CKR(cudaMallocAsync(&yr, (size_t)n_global, st));
    if (c->nccl) {
        CKN(ncclGroupStart());
        for (int r = 0; r < W; ++r) {
            const size_t cnt = (size_t)sz[2 * r + 1] * d;
            CKN(ncclBroadcast(r == c->rank ? (const void*)X_local : nullptr, xr + sz[2 * r] * d, cnt,
                              ncclFloat32, r, c->nccl, st));
            CKN(ncclBroadcast(r == c->rank ? (const void*)y_local : nullptr, yr + sz[2 * r],
                              (size_t)sz[2 * r + 1], ncclInt8, r, c->nccl, st));
        }
        CKN(ncclGroupEnd());
    } else {
        // host bootstrap: every rank's rows (padded to the largest block) through the host
        const size_t rb = (size_t)n_max * d * 4 + (size_t)n_max;
        std::vector<char> mine_b(rb, 0), all_b(rb * W);
        CKR(cudaMemcpyAsync(mine_b.data(), X_local, (size_t)n_local * d * 4, cudaMemcpyDeviceToHost, st));
        CKR(cudaMemcpyAsync(mine_b.data() + (size_t)n_max * d * 4, y_local, (size_t)n_local, cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
        if ((rc = allgather_host(c, mine_b.data(), all_b.data(), rb, st))) { cudaFreeAsync(xr, st); cudaFreeAsync(yr, st); return rc; }
        for (int r = 0; r < W; ++r) {
            CKR(cudaMemcpyAsync(xr + sz[2 * r] * d, all_b.data() + rb * r, (size_t)sz[2 * r + 1] * d * 4,
                                cudaMemcpyHostToDevice, st));
            CKR(cudaMemcpyAsync(yr + sz[2 * r], all_b.data() + rb * r + (size_t)n_max * d * 4, (size_t)sz[2 * r + 1],
                                cudaMemcpyHostToDevice, st));
        }
    }
    rc = validate_device(xr, yr, n_global, d, st, nullptr);
    if (rc) { cudaFreeAsync(xr, st); cudaFreeAsync(yr, st); return rc; }
    // ---- fresh mailboxes on every rank before anyone publishes
    CKR(cudaMemsetAsync(c->mbox_local, 0, c->mbox_bytes, st));
    CKR(cudaStreamSynchronize(st));
    {
        char one = 1;
        std::vector<char> all(W);
        if ((rc = allgather_host(c, &one, all.data(), 1, st))) { cudaFreeAsync(xr, st); cudaFreeAsync(yr, st); return rc; }
    }

    SolveArgs a;
    a.p = p;
    a.n_global = n_global; a.d = d; a.xr = xr;
    // (p.ctas > 0, the same on every rank: fewer CTAs per rank -- e.g. several ranks sharing
    // one device's SMs under MPS; the mailboxes are sized for the full count)
    a.world = W; a.rank_base = c->rank; a.nranks_here = 1;
    a.ctas_per_rank = (p.ctas > 0 && p.ctas < c->ctas_per_rank) ? p.ctas : c->ctas_per_rank;
    a.n_sm = c->n_sm; a.max_smem = c->max_smem;
    for (int r = 0; r < W; ++r) {
        a.row_off[r] = sz[2 * r]; a.n_rows[r] = sz[2 * r + 1];
        if (a.n_rows[r] > a.n_rows_max) a.n_rows_max = a.n_rows[r];
        a.mbox[r] = c->peers[r];
    }
    a.x_rank[c->rank] = xr + row_offset * d;
    a.y_rank[c->rank] = yr + row_offset;
    a.alpha_out[c->rank] = alpha_local;
    a.mbox_local_alloc = false;
    a.stream = st;
    a.timeout_ns = 60ll * 1000 * 1000 * 1000;
    a.alpha0 = dbg ? dbg->alpha0 : nullptr;
    a.f0 = dbg ? dbg->f0 : nullptr;
    a.warm_global = false;
    a.trace = (dbg && c->rank == 0) ? (long long*)dbg->pair_trace : nullptr;
    a.trace_cap = (dbg && c->rank == 0) ? dbg->pair_trace_cap : 0;
    double* f_dev = (dbg && dbg->f_out) ? dbg->f_out : nullptr;
    double* f_tmp = nullptr;
    if (!f_dev) {
        CKR(cudaMallocAsync(&f_tmp, (size_t)(n_local > 0 ? n_local : 1) * 8, st));
        f_dev = f_tmp;
    }
    a.f_out = f_dev; a.f_out_kind = cudaMemcpyDeviceToDevice; a.f_out_global = false;
    rc = solve(a);
    if (rc) { cudaFreeAsync(xr, st); cudaFreeAsync(yr, st); if (f_tmp) cudaFreeAsync(f_tmp, st); return rc; }
    *b = -(a.out.b_up + a.out.b_low) / 2.0;
    if (info) {
        memset(info, 0, sizeof(*info));
        info->iterations = a.out.iterations;
        info->converged = a.out.state == ST_CONVERGED;
        info->b_up = a.out.b_up; info->b_low = a.out.b_low; info->gap = a.out.b_low - a.out.b_up;
        info->seconds_solve = a.out.seconds_solve; info->launches = a.out.launches;
        info->cache_hits = a.out.cache_hits; info->cache_misses = a.out.cache_misses;
        // n_sv and W: per-rank device reductions, summed over ranks in rank order
        double loc[2];
        if ((rc = info_device(alpha_local, f_dev, y_local, n_local, p.sv_epsilon, st, loc))) return rc;
        std::vector<double> all(2 * W);
        if ((rc = allgather_host(c, loc, all.data(), 16, st))) return rc;
        double w = 0.0, nsv = 0.0;
        for (int r = 0; r < W; ++r) { w += all[2 * r]; nsv += all[2 * r + 1]; }
        info->dual_objective = 0.5 * w;
        info->n_sv = (int)nsv;
    }
    CKR(cudaFreeAsync(xr, st));
    CKR(cudaFreeAsync(yr, st));
    if (f_tmp) CKR(cudaFreeAsync(f_tmp, st));
    CKR(cudaStreamSynchronize(st));
    return SVM_OK;
}
