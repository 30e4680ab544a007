// comm.cu -- data-parallel gradient exchange over NCCL (NVLink 5 / NVSwitch).
// The reference has no collectives; this is the exchange step
// of batch-sharded training: a sum all-reduce of the flat gradient buffer in
// buckets on a dedicated comm stream, ordered after the backward kernels that
// produced each bucket (event fork/join with the compute stream, so the whole
// pattern is capturable into the step's CUDA graph).
// NCCL is loaded lazily (dlopen) when the first communicator is created, so
// single-GPU processes never map it and a process that imports torch gets
// torch's bundled NCCL (already loaded, or found next to torch) instead of a
// second, older copy that would shadow torch's symbols.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>

#include "nncb_internal.cuh"

namespace {

struct Nccl {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGetErrorString) getErrorString = nullptr;
    bool ok = false;
    std::string where;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl r;
        std::vector<std::string> candidates;
        if (const char* env = std::getenv("NNCB_NCCL_LIB")) candidates.push_back(env);
        candidates.push_back("libnccl.so.2");   // returns an already-loaded copy first
        void* h = nullptr;
        for (const auto& c : candidates) {
            h = dlopen(c.c_str(), RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
            if (h) {
                r.where = c + " (already loaded)";
                break;
            }
        }
        if (!h)
            for (const auto& c : candidates) {
                h = dlopen(c.c_str(), RTLD_NOW | RTLD_LOCAL);
                if (h) {
                    r.where = c;
                    break;
                }
            }
        if (!h) return r;
        r.getUniqueId = reinterpret_cast<decltype(r.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        r.commInitRank = reinterpret_cast<decltype(r.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        r.commDestroy = reinterpret_cast<decltype(r.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        r.allReduce = reinterpret_cast<decltype(r.allReduce)>(dlsym(h, "ncclAllReduce"));
        r.getErrorString = reinterpret_cast<decltype(r.getErrorString)>(dlsym(h, "ncclGetErrorString"));
        r.ok = r.getUniqueId && r.commInitRank && r.commDestroy && r.allReduce && r.getErrorString;
        return r;
    }();
    return n;
}

}  // namespace

#define NNCB_NCCL(expr)                                                                     \
    do {                                                                                    \
        if (!nccl().ok) return ::nncb::fail("NCCL library could not be loaded");           \
        ncclResult_t _r = (expr);                                                           \
        if (_r != ncclSuccess)                                                              \
            return ::nncb::fail(std::string(#expr) + ": " + nccl().getErrorString(_r));    \
    } while (0)

extern "C" {

int nncb_comm_unique_id(uint8_t id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    NNCB_NCCL(nccl().getUniqueId(&u));
    memcpy(id, &u, 128);
    return 0;
}

int nncb_comm_init(nncb_ctx* ctx, int nranks, int rank, const uint8_t id[128]) {
    if (ctx->nccl_comm) return 0;
    NNCB_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t comm;
    NNCB_NCCL(nccl().commInitRank(&comm, nranks, u, rank));
    ctx->nccl_comm = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return 0;
}

int nncb_comm_destroy(nncb_ctx* ctx) {
    if (!ctx->nccl_comm) return 0;
    if (nccl().ok) nccl().commDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
    ctx->nccl_comm = nullptr;
    return 0;
}

int nncb_allreduce_sum(nncb_ctx* ctx, float* buf, int64_t count) {
    if (!ctx->nccl_comm) return nncb::fail("nncb_allreduce_sum: communicator not initialised");
    if (count <= 0) return 0;
    if (int rc = nncb_allreduce_sum_async(ctx, buf, count)) return rc;
    return nncb_comm_join(ctx);
}

int nncb_allreduce_sum_on_comm(nncb_ctx* ctx, float* buf, int64_t count) {
    if (!ctx->nccl_comm) return nncb::fail("nncb_allreduce_sum_on_comm: communicator not initialised");
    if (count <= 0) return 0;
    NNCB_NCCL(nccl().allReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclSum,
                               static_cast<ncclComm_t>(ctx->nccl_comm), ctx->comm_stream));
    return 0;
}

int nncb_allreduce_sum_async(nncb_ctx* ctx, float* buf, int64_t count) {
    if (!ctx->nccl_comm) return nncb::fail("nncb_allreduce_sum_async: communicator not initialised");
    if (count <= 0) return 0;
    if (int rc = nncb_fork(ctx, NNCB_STREAM_COMM)) return rc;
    return nncb_allreduce_sum_on_comm(ctx, buf, count);
}

int nncb_comm_join(nncb_ctx* ctx) { return nncb_join(ctx, NNCB_STREAM_COMM); }

int nncb_comm_active(nncb_ctx* ctx) { return ctx->nccl_comm ? 1 : 0; }

}  // extern "C"
