// comm.cu -- one process per GPU: communicator, peer mailboxes, svm_train_shard.
//
// The per-iteration exchange is device-initiated inside the
// persistent kernel: every CTA stores its 48-byte candidate record into every rank's
// mailbox through NVLink peer pointers and bumps that rank's arrival counter with a
// system-scope atomic.  NCCL is used only for setup (bootstrap, the one-time allgather
// of the row-major X replica used to gather the two pivot rows, IPC handles, and the
// final dual-objective sum).
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
    CKR(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    int rc = device_limits(&c->n_sm, &c->max_smem);
    if (rc) return rc;
    // agree on the CTA count per rank (minimum SM count over ranks)
    int* dv;
    CKR(cudaMalloc(&dv, 4));
    CKR(cudaMemcpy(dv, &c->n_sm, 4, cudaMemcpyHostToDevice));
    CKN(ncclAllReduce(dv, dv, 1, ncclInt32, ncclMin, c->nccl, c->st));
    CKR(cudaMemcpyAsync(&c->ctas_per_rank, dv, 4, cudaMemcpyDeviceToHost, c->st));
    CKR(cudaStreamSynchronize(c->st));
    cudaFree(dv);
    // mailbox + peer mapping
    c->mbox_bytes = svmk::mbox_bytes(c->ctas_per_rank, world);
    CKR(cudaMalloc(&c->mbox_local, c->mbox_bytes));
    CKR(cudaMemset(c->mbox_local, 0, c->mbox_bytes));
    cudaIpcMemHandle_t h;
    CKR(cudaIpcGetMemHandle(&h, c->mbox_local));
    char* dh;
    CKR(cudaMalloc(&dh, sizeof(h) * world));
    CKR(cudaMemcpy(dh + sizeof(h) * rank, &h, sizeof(h), cudaMemcpyHostToDevice));
    CKN(ncclAllGather(dh + sizeof(h) * rank, dh, sizeof(h), ncclChar, c->nccl, c->st));
    std::vector<cudaIpcMemHandle_t> all(world);
    CKR(cudaMemcpyAsync(all.data(), dh, sizeof(h) * world, cudaMemcpyDeviceToHost, c->st));
    CKR(cudaStreamSynchronize(c->st));
    cudaFree(dh);
    for (int r = 0; r < world; ++r) {
        if (r == rank) { c->peers[r] = c->mbox_local; continue; }
        void* ptr = nullptr;
        CKR(cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess));
        c->peers[r] = (Mailbox*)ptr;
    }
    *out = c;
    return SVM_OK;
}

extern "C" void svm_comm_destroy(void* comm) {
    Comm* c = (Comm*)comm;
    if (!c) return;
    cudaSetDevice(c->device);
    for (int r = 0; r < c->world; ++r)
        if (r != c->rank && c->peers[r]) cudaIpcCloseMemHandle(c->peers[r]);
    if (c->mbox_local) cudaFree(c->mbox_local);
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

extern "C" int svm_train_shard(void* comm, const float* X_local, const int8_t* y_local,
                               int64_t n_local, int64_t row_offset, int64_t n_global, int64_t d,
                               const svm_params* p_in, double* alpha_local, double* b,
                               svm_info* info, void* cuda_stream) {
    Comm* c = (Comm*)comm;
    if (!c || !X_local || !y_local || !alpha_local || !b) return fail(SVM_EINVAL, "null pointer");
    svm_params p;
    int rc = check_params(n_global, d, p_in, &p);
    if (rc) return rc;
    if (n_local < 0 || row_offset < 0 || row_offset + n_local > n_global)
        return fail(SVM_EINVAL, "row block outside [0, n_global)");
    cudaStream_t st = cuda_stream ? (cudaStream_t)cuda_stream : c->st;
    CKR(cudaSetDevice(c->device));
    const int W = c->world;
    // ---- every rank's (row_offset, n_local)
    long long* dsz;
    CKR(cudaMallocAsync(&dsz, 16 * W, st));
    long long mine[2] = {row_offset, n_local};
    CKR(cudaMemcpyAsync(dsz + 2 * c->rank, mine, 16, cudaMemcpyHostToDevice, st));
    CKN(ncclAllGather(dsz + 2 * c->rank, dsz, 2, ncclInt64, c->nccl, st));
    std::vector<long long> sz(2 * W);
    CKR(cudaMemcpyAsync(sz.data(), dsz, 16 * W, cudaMemcpyDeviceToHost, st));
    CKR(cudaFreeAsync(dsz, st));
    CKR(cudaStreamSynchronize(st));
    long long covered = 0;
    for (int r = 0; r < W; ++r) {
        if (sz[2 * r] != covered) return fail(SVM_EINVAL, "row blocks must be contiguous in rank order");
        covered += sz[2 * r + 1];
    }
    if (covered != n_global) return fail(SVM_EINVAL, "row blocks do not cover n_global");
    // ---- the row-major replica of X (pivot rows are gathered from it) and y
    float* xr;
    int8_t* yr;
    CKR(cudaMallocAsync(&xr, (size_t)n_global * d * 4, st));
    CKR(cudaMallocAsync(&yr, (size_t)n_global, st));
    CKN(ncclGroupStart());
    for (int r = 0; r < W; ++r) {
        const size_t cnt = (size_t)sz[2 * r + 1] * d;
        CKN(ncclBroadcast(r == c->rank ? (const void*)X_local : nullptr, xr + sz[2 * r] * d, cnt,
                          ncclFloat32, r, c->nccl, st));
        CKN(ncclBroadcast(r == c->rank ? (const void*)y_local : nullptr, yr + sz[2 * r],
                          (size_t)sz[2 * r + 1], ncclInt8, r, c->nccl, st));
    }
    CKN(ncclGroupEnd());
    rc = validate_device(xr, yr, n_global, d, st, nullptr);
    if (rc) { cudaFreeAsync(xr, st); cudaFreeAsync(yr, st); return rc; }
    // ---- fresh mailboxes on every rank before anyone publishes
    CKR(cudaMemsetAsync(c->mbox_local, 0, c->mbox_bytes, st));
    int* dummy;
    CKR(cudaMallocAsync(&dummy, 4, st));
    CKN(ncclAllReduce(dummy, dummy, 1, ncclInt32, ncclSum, c->nccl, st));
    CKR(cudaFreeAsync(dummy, st));
    CKR(cudaStreamSynchronize(st));

    SolveArgs a;
    a.p = p;
    a.n_global = n_global; a.d = d; a.xr = xr;
    a.world = W; a.rank_base = c->rank; a.nranks_here = 1; a.ctas_per_rank = c->ctas_per_rank;
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
    double* f_dev;
    CKR(cudaMallocAsync(&f_dev, (size_t)(n_local > 0 ? n_local : 1) * 8, st));
    a.f_out = f_dev; a.f_out_kind = cudaMemcpyDeviceToDevice; a.f_out_global = false;
    rc = solve(a);
    if (rc) { cudaFreeAsync(xr, st); cudaFreeAsync(yr, st); cudaFreeAsync(f_dev, st); return rc; }
    *b = -(a.out.b_up + a.out.b_low) / 2.0;
    if (info) {
        memset(info, 0, sizeof(*info));
        info->iterations = a.out.iterations;
        info->converged = a.out.state == ST_CONVERGED;
        info->b_up = a.out.b_up; info->b_low = a.out.b_low; info->gap = a.out.b_low - a.out.b_up;
        info->seconds_solve = a.out.seconds_solve; info->launches = a.out.launches;
        std::vector<double> ha((size_t)n_local), hf((size_t)n_local);
        std::vector<int8_t> hy((size_t)n_local);
        CKR(cudaMemcpyAsync(ha.data(), alpha_local, (size_t)n_local * 8, cudaMemcpyDeviceToHost, st));
        CKR(cudaMemcpyAsync(hf.data(), f_dev, (size_t)n_local * 8, cudaMemcpyDeviceToHost, st));
        CKR(cudaMemcpyAsync(hy.data(), y_local, (size_t)n_local, cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
        double loc[2] = {0.0, 0.0};
        for (long long j = 0; j < n_local; ++j) {
            loc[0] += ha[j] * (1.0 - (double)hy[j] * hf[j]);
            loc[1] += ha[j] > p.sv_epsilon;
        }
        double* dl;
        CKR(cudaMallocAsync(&dl, 16, st));
        CKR(cudaMemcpyAsync(dl, loc, 16, cudaMemcpyHostToDevice, st));
        CKN(ncclAllReduce(dl, dl, 2, ncclFloat64, ncclSum, c->nccl, st));
        CKR(cudaMemcpyAsync(loc, dl, 16, cudaMemcpyDeviceToHost, st));
        CKR(cudaFreeAsync(dl, st));
        CKR(cudaStreamSynchronize(st));
        info->dual_objective = 0.5 * loc[0];
        info->n_sv = (int)loc[1];
    }
    CKR(cudaFreeAsync(xr, st));
    CKR(cudaFreeAsync(yr, st));
    CKR(cudaFreeAsync(f_dev, st));
    CKR(cudaStreamSynchronize(st));
    return SVM_OK;
}
