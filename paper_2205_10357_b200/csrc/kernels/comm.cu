// comm.cu -- data-parallel gradient exchange over NCCL (NVLink 5 / NVSwitch).
// The reference has no collectives; this is the exchange step
// of batch-sharded training: a sum all-reduce of the flat gradient buffer in
// buckets on a dedicated comm stream, ordered after the backward kernels that
// produced each bucket (event fork/join with the compute stream, so the whole
// pattern is capturable into the step's CUDA graph).
#include <nccl.h>

#include "nncb_internal.cuh"

#define NNCB_NCCL(expr)                                                                     \
    do {                                                                                    \
        ncclResult_t _r = (expr);                                                           \
        if (_r != ncclSuccess)                                                              \
            return ::nncb::fail(std::string(#expr) + ": " + ncclGetErrorString(_r));       \
    } while (0)

extern "C" {

int nncb_comm_unique_id(uint8_t id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    NNCB_NCCL(ncclGetUniqueId(&u));
    memcpy(id, &u, 128);
    return 0;
}

int nncb_comm_init(nncb_ctx* ctx, int nranks, int rank, const uint8_t id[128]) {
    if (ctx->nccl_comm) return 0;
    NNCB_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t comm;
    NNCB_NCCL(ncclCommInitRank(&comm, nranks, u, rank));
    ctx->nccl_comm = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return 0;
}

int nncb_comm_destroy(nncb_ctx* ctx) {
    if (!ctx->nccl_comm) return 0;
    ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
    ctx->nccl_comm = nullptr;
    return 0;
}

int nncb_allreduce_sum(nncb_ctx* ctx, float* buf, int64_t count) {
    if (!ctx->nccl_comm) return nncb::fail("nncb_allreduce_sum: communicator not initialised");
    if (count <= 0) return 0;
    cudaEvent_t ready, done;
    NNCB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    NNCB_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    NNCB_CUDA(cudaEventRecord(ready, ctx->stream));
    NNCB_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ready, 0));
    NNCB_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclSum,
                            static_cast<ncclComm_t>(ctx->nccl_comm), ctx->comm_stream));
    NNCB_CUDA(cudaEventRecord(done, ctx->comm_stream));
    NNCB_CUDA(cudaStreamWaitEvent(ctx->stream, done, 0));
    cudaEventDestroy(ready);
    cudaEventDestroy(done);
    return 0;
}

}  // extern "C"
