// nncb_core.cu -- context, device memory, streams, CUDA graphs, events.
// Replaces the reference's host-side ExecutionContext byte store
// (runtime.cpp:108-152) and OffloadDevice transfers (runtime.cpp:71-102).
#include <cstdio>
#include <cstring>

#include "nncb_internal.cuh"

namespace nncb {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }
int fail(const std::string& msg) {
    g_error = msg;
    return 1;
}

void* scratch(nncb_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->scratch_bytes) return ctx->scratch;
    if (ctx->scratch) ctx->retired.push_back(ctx->scratch);
    size_t want = bytes < (1u << 20) ? (1u << 20) : bytes;
    if (cudaMalloc(&ctx->scratch, want) != cudaSuccess) {
        ctx->scratch = nullptr;
        ctx->scratch_bytes = 0;
        return nullptr;
    }
    ctx->scratch_bytes = want;
    return ctx->scratch;
}

void* wt_buffer(nncb_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->wt_bytes) return ctx->wt;
    if (ctx->wt) ctx->retired.push_back(ctx->wt);   // captured graphs may still reference it
    if (cudaMalloc(&ctx->wt, bytes) != cudaSuccess) {
        ctx->wt = nullptr;
        ctx->wt_bytes = 0;
        return nullptr;
    }
    ctx->wt_bytes = bytes;
    return ctx->wt;
}

void* bf16_buffer(nncb_ctx* ctx, int which, size_t bytes) {
    if (bytes <= ctx->bf16_bytes[which]) return ctx->bf16_buf[which];
    if (ctx->bf16_buf[which]) ctx->retired.push_back(ctx->bf16_buf[which]);   // captured graphs may use it
    if (cudaMalloc(&ctx->bf16_buf[which], bytes) != cudaSuccess) {
        ctx->bf16_buf[which] = nullptr;
        ctx->bf16_bytes[which] = 0;
        return nullptr;
    }
    ctx->bf16_bytes[which] = bytes;
    return ctx->bf16_buf[which];
}

void* bn_inv_buffer(nncb_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->bn_inv_bytes) return ctx->bn_inv;
    if (ctx->bn_inv) ctx->retired.push_back(ctx->bn_inv);
    const size_t want = bytes < 65536 ? 65536 : bytes;
    if (cudaMalloc(&ctx->bn_inv, want) != cudaSuccess) {
        ctx->bn_inv = nullptr;
        ctx->bn_inv_bytes = 0;
        return nullptr;
    }
    ctx->bn_inv_bytes = want;
    return ctx->bn_inv;
}

void* colstats_fixed_buffer(nncb_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->cs_fixed_bytes) return ctx->cs_fixed;
    if (ctx->cs_fixed) ctx->retired.push_back(ctx->cs_fixed);   // captured graphs may use it
    const size_t want = bytes < (1u << 16) ? (1u << 16) : bytes;
    if (cudaMalloc(&ctx->cs_fixed, want) != cudaSuccess) {
        ctx->cs_fixed = nullptr;
        ctx->cs_fixed_bytes = 0;
        return nullptr;
    }
    ctx->cs_fixed_bytes = want;
    return ctx->cs_fixed;
}

void* workspace(nncb_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->workspace_bytes) return ctx->workspace;
    if (ctx->workspace) ctx->retired.push_back(ctx->workspace);
    ctx->s2d_src = nullptr;   // a lowered input in the old workspace is not carried over
    if (cudaMalloc(&ctx->workspace, bytes) != cudaSuccess) {
        ctx->workspace = nullptr;
        ctx->workspace_bytes = 0;
        return nullptr;
    }
    ctx->workspace_bytes = bytes;
    return ctx->workspace;
}

}  // namespace nncb

using nncb::fail;

namespace nncb {
cudaEvent_t fork_event(nncb_ctx* ctx) {
    cudaEvent_t e = ctx->fork_events[ctx->fork_next];
    ctx->fork_next = (ctx->fork_next + 1) % ctx->fork_events.size();
    return e;
}
cudaStream_t stream_of(nncb_ctx* ctx, int id) {
    return id == NNCB_STREAM_COPY ? ctx->copy_stream : id == NNCB_STREAM_COMM ? ctx->comm_stream : ctx->stream;
}
}  // namespace nncb

extern "C" {

const char* nncb_last_error(void) { return nncb::g_error.c_str(); }

int nncb_create(int device, nncb_ctx** out) {
    int count = 0;
    NNCB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail("nncb_create: no CUDA device " + std::to_string(device));
    NNCB_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    NNCB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail("nncb_create: this build targets sm_100a (B200); device " + std::string(prop.name) +
                    " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
    auto* c = new nncb_ctx;
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    NNCB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    NNCB_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    NNCB_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    c->fork_events.resize(256);
    for (auto& e : c->fork_events) NNCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *out = c;
    return 0;
}

int nncb_destroy(nncb_ctx* c) {
    if (!c) return 0;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->copy_stream);
    nncb_comm_destroy(c);
    for (auto& [k, v] : c->ew_cache) {
        (void)k;
        nncb::ew_release(v);
    }
    nncb::staging_release(c);
    if (c->scratch) cudaFree(c->scratch);
    for (void* p : c->retired) cudaFree(p);
    if (c->workspace) cudaFree(c->workspace);
    if (c->wt) cudaFree(c->wt);
    for (void* p : c->bf16_buf)
        if (p) cudaFree(p);
    if (c->bn_inv) cudaFree(c->bn_inv);
    if (c->cs_fixed) cudaFree(c->cs_fixed);
    cudaStreamSynchronize(c->comm_stream);
    for (cudaEvent_t e : c->fork_events) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->comm_stream);
    cudaStreamDestroy(c->copy_stream);
    delete c;
    return 0;
}

int nncb_device_info(nncb_ctx* c, int* sms, int* major, int* minor, size_t* total) {
    cudaDeviceProp prop;
    NNCB_CUDA(cudaGetDeviceProperties(&prop, c->device));
    if (sms) *sms = prop.multiProcessorCount;
    if (major) *major = prop.major;
    if (minor) *minor = prop.minor;
    if (total) *total = prop.totalGlobalMem;
    return 0;
}

int nncb_malloc(nncb_ctx* c, size_t bytes, void** out) {
    NNCB_CUDA(cudaSetDevice(c->device));
    *out = nullptr;
    if (bytes == 0) return 0;
    NNCB_CUDA(cudaMalloc(out, bytes));
    return 0;
}

int nncb_free(nncb_ctx* c, void* p) {
    if (!p) return 0;
    NNCB_CUDA(cudaSetDevice(c->device));
    NNCB_CUDA(cudaFree(p));
    return 0;
}

int nncb_host_alloc(size_t bytes, void** out) {
    NNCB_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
    return 0;
}

int nncb_host_free(void* p) {
    if (p) NNCB_CUDA(cudaFreeHost(p));
    return 0;
}

int nncb_memset(nncb_ctx* c, void* dst, int v, size_t bytes) {
    if (bytes) NNCB_CUDA(cudaMemsetAsync(dst, v, bytes, c->stream));
    return 0;
}

int nncb_d2d(nncb_ctx* c, void* dst, const void* src, size_t bytes) {
    if (bytes) NNCB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
    return 0;
}

int nncb_sync(nncb_ctx* c) {
    NNCB_CUDA(cudaStreamSynchronize(c->stream));
    NNCB_CUDA(cudaGetLastError());
    return 0;
}

void* nncb_stream(nncb_ctx* c) { return c->stream; }

int nncb_capture_begin(nncb_ctx* c) {
    NNCB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    return 0;
}

int nncb_capture_end(nncb_ctx* c, void** exec) {
    cudaGraph_t graph = nullptr;
    NNCB_CUDA(cudaStreamEndCapture(c->stream, &graph));
    cudaGraphExec_t ge = nullptr;
    cudaError_t e = cudaGraphInstantiate(&ge, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    *exec = ge;
    return 0;
}

int nncb_graph_launch(nncb_ctx* c, void* exec) {
    NNCB_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), c->stream));
    return 0;
}

int nncb_graph_destroy(void* exec) {
    if (exec) NNCB_CUDA(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec)));
    return 0;
}

int nncb_event_create(void** ev) {
    cudaEvent_t e;
    NNCB_CUDA(cudaEventCreate(&e));
    *ev = e;
    return 0;
}

int nncb_event_record(nncb_ctx* c, void* ev) {
    NNCB_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), c->stream));
    return 0;
}

int nncb_event_record_on(nncb_ctx* c, int stream, void* ev) {
    NNCB_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), nncb::stream_of(c, stream)));
    return 0;
}

int nncb_stream_wait(nncb_ctx* c, int stream, void* ev) {
    NNCB_CUDA(cudaStreamWaitEvent(nncb::stream_of(c, stream), static_cast<cudaEvent_t>(ev), 0));
    return 0;
}

int nncb_fork(nncb_ctx* c, int to_stream) {
    cudaEvent_t e = nncb::fork_event(c);
    NNCB_CUDA(cudaEventRecord(e, c->stream));
    NNCB_CUDA(cudaStreamWaitEvent(nncb::stream_of(c, to_stream), e, 0));
    return 0;
}

int nncb_join(nncb_ctx* c, int from_stream) {
    cudaEvent_t e = nncb::fork_event(c);
    NNCB_CUDA(cudaEventRecord(e, nncb::stream_of(c, from_stream)));
    NNCB_CUDA(cudaStreamWaitEvent(c->stream, e, 0));
    return 0;
}

int nncb_set_f64(nncb_ctx* c, double* dst, double value) {
    // stream-ordered 8-byte write (the pageable source is staged by the driver
    // before the call returns); never called during a capture
    NNCB_CUDA(cudaMemcpyAsync(dst, &value, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    return 0;
}

int nncb_event_sync(void* ev) {
    NNCB_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(ev)));
    return 0;
}

int nncb_event_elapsed_ms(void* a, void* b, float* ms) {
    NNCB_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(b)));
    NNCB_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)));
    return 0;
}

int nncb_event_destroy(void* ev) {
    if (ev) NNCB_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
    return 0;
}

uint64_t nncb_launch_count(nncb_ctx* c) { return c->launches.load(); }

}  // extern "C"
