// nncb_internal.cuh -- shared internals of libnncb.so (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "nncb.h"

struct nncb_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;       // compute stream
    cudaStream_t comm_stream = nullptr;  // collectives
    cudaStream_t copy_stream = nullptr;  // pipelined input uploads (nncb_h2d_async)
    std::atomic<uint64_t> launches{0};
    void* nccl_comm = nullptr;
    int nranks = 1, rank = 0;
    // fused-kernel cache: program hash -> kernel
    std::map<std::string, nncb_ew_kernel*> ew_cache;
    // scratch for reductions (grid partials), grown on demand
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    std::vector<void*> retired;          // outgrown scratch kept alive (captured graphs may use it)
    void* workspace = nullptr;           // im2col columns (separate from reduction scratch)
    size_t workspace_bytes = 0;
    // the space-to-depth input most recently lowered into `workspace` (stream
    // order): source, geometry and the workspace it lives in (NNCB_EPI_A_UNCHANGED)
    const void* s2d_src = nullptr;
    int64_t s2d_key[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    void* s2d_ws = nullptr;
    void* staging = nullptr;             // pinned upload ring (host_io.cu), created on first large h2d
    void* wt = nullptr;                  // transposed (K-major) forward weights, grown on demand
    size_t wt_bytes = 0;
    void* bf16_buf[2] = {nullptr, nullptr};   // bf16 operand copies of a NNCB_PREC_BF16 GEMM (A, B)
    size_t bf16_bytes[2] = {0, 0};
    void* bn_inv = nullptr;              // per-call invstd of a BN_AFFINE epilogue
    size_t bn_inv_bytes = 0;
    void* cs_fixed = nullptr;            // fixed-point column-statistics accumulators of a GEMM epilogue
    size_t cs_fixed_bytes = 0;
    // fork/join events between the compute and comm streams, reused round
    // robin (created once: nothing is created or destroyed during a capture)
    std::vector<cudaEvent_t> fork_events;
    size_t fork_next = 0;
};

namespace nncb {

// Programmatic dependent launch of a small follow-up kernel (finalize, fold):
// it may be scheduled while the preceding grid drains and must begin with
// pdl_wait() (griddepcontrol.wait: the preceding grid is complete and its
// memory visible past that point).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }


void set_error(const std::string& msg);
/// The next event of the context's fork/join pool.
cudaEvent_t fork_event(nncb_ctx* ctx);
cudaStream_t stream_of(nncb_ctx* ctx, int id);
void staging_release(nncb_ctx* c);
void* wt_buffer(nncb_ctx* ctx, size_t bytes);
int fail(const std::string& msg);

#define NNCB_CUDA(expr)                                                                       \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess) {                                                              \
            cudaGetLastError(); /* clear non-sticky errors so later calls report their own */ \
            return ::nncb::fail(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" +   \
                                __FILE__ + ":" + std::to_string(__LINE__) + ")");            \
        }                                                                                     \
    } while (0)

#define NNCB_LAUNCHED(ctx)                                                                    \
    do {                                                                                      \
        cudaError_t _e = cudaGetLastError();                                                  \
        if (_e != cudaSuccess)                                                                \
            return ::nncb::fail(std::string("launch failed: ") + cudaGetErrorString(_e) +     \
                                " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")");     \
        (ctx)->launches.fetch_add(1, std::memory_order_relaxed);                              \
    } while (0)

/// Grid-stride sizing: a multiple of the SM count (resident CTAs per SM x SMs).
inline unsigned grid_for(const nncb_ctx* ctx, int64_t work_items, int threads, int per_sm = 8) {
    int64_t want = (work_items + threads - 1) / threads;
    int64_t cap = static_cast<int64_t>(ctx->sm_count) * per_sm;
    if (want < 1) want = 1;
    return static_cast<unsigned>(want < cap ? want : cap);
}

void* scratch(nncb_ctx* ctx, size_t bytes);
void* bf16_buffer(nncb_ctx* ctx, int which, size_t bytes);
void* bn_inv_buffer(nncb_ctx* ctx, size_t bytes);
void* colstats_fixed_buffer(nncb_ctx* ctx, size_t bytes);
int affine_relu_output(nncb_ctx* ctx, const nncb_gemm_desc* d, float* out);
void* workspace(nncb_ctx* ctx, size_t bytes);
void ew_release(nncb_ew_kernel* k);

int colstats_from_output(nncb_ctx* ctx, const float* y, double* cs, int64_t rows, int64_t C);

// GEMM back ends (gemm_simt.cu / gemm_tc.cu)
int gemm_simt(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
              float* out);
int gemm_tc(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
            float* out, bool* handled);
// whether the last weight-gradient GEMM on this thread applied its fused SGD
// update (and clears the flag)
bool take_sgd_applied();
// NNCB_PREC_TF32X3: split operands, tf32 GEMM over the K-concatenated problem
int gemm_tc_x3(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
               float* out, bool* handled);

}  // namespace nncb
