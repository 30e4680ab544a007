/* include/nncb.h -- thin C-ABI of the B200 kernel layer (libnncb.so).
 *
 * The reference has no device layer: every kernel is a C++ template in
 * core/include/nnc/kernels.hpp run on the host by runtime::execute
 * (core/src/runtime.cpp:160-306). This header is the sm_100a replacement of
 * that kernel set, called by the C++ host (libnnc_b200.so) -- never by users
 * directly. Plain C: int status (0 = OK), nncb_last_error(), no exceptions,
 * no torch types. One nncb_ctx per GPU, used by one host thread at a time.
 * All launches are asynchronous on the context's compute stream.
 *
 * Which reference routine each entry point replaces is cited per function.
 */
#ifndef NNCB_H
#define NNCB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nncb_ctx nncb_ctx;
typedef struct nncb_ew_kernel nncb_ew_kernel;

/* ------------------------------------------------------------------ */
/*  Context, memory, streams (replaces ExecutionContext's host buffers, */
/*  runtime.hpp:92-121, and OffloadDevice's byte store, runtime.hpp:47-75) */
/* ------------------------------------------------------------------ */
int         nncb_create(int device_ordinal, nncb_ctx** out);
int         nncb_destroy(nncb_ctx* ctx);
const char* nncb_last_error(void);
int         nncb_device_info(nncb_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor,
                             size_t* total_mem);
int         nncb_malloc(nncb_ctx* ctx, size_t bytes, void** out);
int         nncb_free(nncb_ctx* ctx, void* ptr);
int         nncb_host_alloc(size_t bytes, void** out);        /* pinned host memory */
int         nncb_host_free(void* ptr);
int         nncb_memset(nncb_ctx* ctx, void* dst, int value, size_t bytes);
int         nncb_h2d(nncb_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Parallel host memcpy on the library's copy threads (host staging helper). */
int         nncb_host_copy(void* dst, const void* src, size_t bytes);
int         nncb_d2h(nncb_ctx* ctx, void* dst, const void* src, size_t bytes);
int         nncb_d2d(nncb_ctx* ctx, void* dst, const void* src, size_t bytes);
int         nncb_sync(nncb_ctx* ctx);
void*       nncb_stream(nncb_ctx* ctx);                       /* cudaStream_t */

/* CUDA-graph capture of a launch sequence (one graph per bound plan). */
int nncb_capture_begin(nncb_ctx* ctx);
int nncb_capture_end(nncb_ctx* ctx, void** graph_exec);
int nncb_graph_launch(nncb_ctx* ctx, void* graph_exec);
int nncb_graph_destroy(void* graph_exec);

/* Device-side timing on the compute stream. */
int nncb_event_create(void** ev);
int nncb_event_record(nncb_ctx* ctx, void* ev);
int nncb_event_elapsed_ms(void* start, void* stop, float* ms);
int nncb_event_destroy(void* ev);

/* Input pipelining: uploads on the context's copy stream overlap the compute
 * stream. nncb_h2d_async returns once the host bytes are handed to DMA (a
 * pageable source is first copied into the pinned ring by the copy threads),
 * so `src` may be reused on return; the device bytes are valid after the
 * copy stream reaches that point (nncb_event_record_on / nncb_stream_wait). */
enum nncb_stream_id { NNCB_STREAM_COMPUTE = 0, NNCB_STREAM_COPY = 1, NNCB_STREAM_COMM = 2 };
int nncb_h2d_async(nncb_ctx* ctx, void* dst, const void* src, size_t bytes);
int nncb_d2h_async(nncb_ctx* ctx, void* dst_pinned, const void* src, size_t bytes);   /* compute stream */
int nncb_event_record_on(nncb_ctx* ctx, int stream, void* ev);
int nncb_stream_wait(nncb_ctx* ctx, int stream, void* ev);
int nncb_event_sync(void* ev);
/* Fork/join between the compute stream and another context stream (pooled
 * events, safe inside a capture): nncb_fork makes `to_stream` wait for the
 * compute stream's current position; nncb_join makes the compute stream wait
 * for everything issued on `from_stream` so far.                            */
int nncb_fork(nncb_ctx* ctx, int to_stream);
int nncb_join(nncb_ctx* ctx, int from_stream);
/* Stream-ordered write of one double (e.g. the learning rate a captured step
 * graph reads; not for use during a capture).                              */
int nncb_set_f64(nncb_ctx* ctx, double* dst_dev, double value);

/* Number of nncb kernel launches issued on this context (all families). */
uint64_t nncb_launch_count(nncb_ctx* ctx);

/* ------------------------------------------------------------------ */
/*  Fused elementwise group: replaces run_ew (runtime.cpp:280-306) and  */
/*  the per-element REF kernels relu/relu_grad/add/mul/copy            */
/*  (kernels.hpp:47-70). The program is compiled once to a dedicated   */
/*  sm_100a kernel (NVRTC) and launched with one pointer per slot.      */
/* ------------------------------------------------------------------ */
enum nncb_ew_op {
    NNCB_EW_LOAD = 0,       /* r[dst] = slot[s][i]                 (mode: element)      */
    NNCB_EW_LOAD_CH = 1,    /* r[dst] = slot[s][i % C]             (per-channel param)  */
    NNCB_EW_STORE = 2,      /* slot[s][i] = r[a]                                        */
    NNCB_EW_RELU = 3,       /* r[dst] = r[a] > 0 ? r[a] : 0  (kernels.hpp:47-50)        */
    NNCB_EW_RELU_GRAD = 4,  /* r[dst] = r[a] > 0 ? r[b] : 0  (kernels.hpp:52-55)        */
    NNCB_EW_ADD = 5,        /* r[dst] = r[a] + r[b]  (round-to-nearest, no FMA)         */
    NNCB_EW_MUL = 6,        /* r[dst] = r[a] * r[b]                                     */
    NNCB_EW_COPY = 7,       /* r[dst] = r[a]                                            */
    NNCB_EW_BN_APPLY = 8,   /* r[dst] = ((r[a]-mean)*invstd)*gamma + beta; operands:
                               b = mean reg, c = invstd reg, d = gamma reg, e = beta reg  */
    NNCB_EW_GELU = 9,       /* r[dst] = 0.5*x*(1+erf(x/sqrt2)) computed in double        */
    NNCB_EW_GELU_GRAD = 10, /* r[dst] = g*(Phi(x) + x*phi(x)), a = x, b = g, in double   */
    NNCB_EW_BN_GRAD = 11,   /* dx = (gamma*invstd) * (g - (sum_g + xhat*sum_gx)/M)
                               a = x, b = g, c = mean, d = invstd, e = gamma,
                               f = sum_g reg, h = sum_gx reg; imm = M (count)            */
    NNCB_EW_BN_INFER = 12,  /* inference BatchNorm from moving statistics:
                               invstd = (float)(1/sqrt((double)var + imm));
                               r[dst] = ((x - mean)*invstd)*gamma + beta;
                               a = x, b = mean, c = var, d = gamma, e = beta         */
    NNCB_EW_BN_GRAD_FAST = 14, /* BN_GRAD operands, per-channel quotients instead of a per-element
                               division: dx = (gamma*invstd) * ((g - sum_g/M) - xhat*(sum_gx/M)).
                               Not bit-identical to BN_GRAD; the runtime uses it only in the
                               tf32 precision mode.                                       */
    NNCB_EW_GELU_FAST = 15,      /* GELU in fp32 (erff): tf32 precision mode only            */
    NNCB_EW_GELU_GRAD_FAST = 16, /* GELU gradient in fp32 (erff/expf): tf32 precision mode only */
    NNCB_EW_REDUCE_STATS = 17,   /* BatchNorm training statistics of r[a] computed inside a
                               fused pass (the group's chain recomputed up to the BN input,
                               nothing stored): per channel sum v and sum v^2 in double,
                               finalized to slot[s][0:C] = mean, slot[s][C:2C] =
                               1/sqrt(var + imm) (biased variance), imm = eps. Same
                               channel-stationary launch requirements as REDUCE_BN_GRAD;
                               counts toward its at-most-two reductions per program.      */
    NNCB_EW_REDUCE_BN_GRAD = 13, /* BatchNorm backward reduction fused into the group that
                               produces g (replaces nncb_bn_grad_reduce for it):
                               sum_g[c] += g, sum_gx[c] += g*xhat, xhat = (x-mean)*invstd,
                               accumulated in double per channel. a = g, b = x,
                               c = mean, d = invstd (LOAD_CH regs); outputs: slot = sum_g,
                               e = sum_gx slot index. Needs the channel-stationary launch:
                               C a power of two in [4, 8192], n % 4 == 0, 16 B-aligned
                               slots; at most two per program (e.g. the two BatchNorms
                               of a residual join fed the same gradient).                */
    NNCB_EW_REDUCE_SUM = 18,     /* per-channel column sum of r[a] in double into the float
                               [C] slot `slot` (a Dense bias gradient folded into the group
                               that stores the gradient). Channel-stationary launch with C
                               a power of two in [4, 8192]; counts toward the at-most-two
                               reductions per program.                                    */
};

typedef struct {
    int32_t op;
    int32_t dst, a, b, c, d, e, f, h;
    int32_t slot;
    double imm;
} nncb_ew_instr;

typedef struct {
    int32_t n_instr;
    const nncb_ew_instr* instr;
    int32_t n_regs;
    int32_t n_slots;
} nncb_ew_program;

int nncb_ew_compile(nncb_ctx* ctx, const nncb_ew_program* prog, nncb_ew_kernel** out);
/* n = element count of the group's iteration space, channels = C for LOAD_CH. */
int nncb_ew_launch(nncb_ctx* ctx, nncb_ew_kernel* k, void* const* slots, int64_t n,
                   int64_t channels);
/* Generates and NVRTC-compiles a program without a device (build-time check). */
int nncb_ew_compile_check(const nncb_ew_program* prog);
/* Generated CUDA source of a compiled program (for inspection / profiles). */
const char* nncb_ew_source(nncb_ew_kernel* k);

/* ------------------------------------------------------------------ */
/*  Tensor-core GEMMs: replace dense/dense_tiled/dense_grad_* and      */
/*  conv2d/conv2d_tiled/conv2d_grad_* (kernels.hpp:118-243, 354-418).  */
/* ------------------------------------------------------------------ */
enum nncb_gemm_kind {
    NNCB_DENSE_FWD = 0,    /* y[b,o]  = bias[o] + sum_i x[b,i] w[i,o]       kernels.hpp:118-127 */
    NNCB_DENSE_DGRAD = 1,  /* gx[b,i] = sum_o g[b,o] w[i,o]                 kernels.hpp:130-139 */
    NNCB_DENSE_WGRAD = 2,  /* gw[i,o] = sum_b x[b,i] g[b,o]                 kernels.hpp:142-151 */
    NNCB_CONV_FWD = 3,     /* NHWC conv, kernel [kh,kw,ci,co], TF-SAME      kernels.hpp:166-190 */
    NNCB_CONV_DGRAD = 4,   /* transposed correlation                        kernels.hpp:192-218 */
    NNCB_CONV_WGRAD = 5,   /* gk[dh,dw,ci,co] = sum x*g                      kernels.hpp:220-243 */
};
enum nncb_precision {
    NNCB_PREC_TF32 = 0,    /* tcgen05.mma kind::tf32, fp32 accumulate in TMEM (default)    */
    NNCB_PREC_FP32 = 1,    /* exact-order fp32 FFMA path (parity mode)                      */
    NNCB_PREC_BF16 = 2,    /* tcgen05.mma kind::f16 on bf16 operands, fp32 accumulate in TMEM:
                              the forward and input-gradient contractions (conv and dense)
                              with K-major operands (conv: channels per tap % 64 == 0, or a
                              single tap with K % 8 == 0) convert A and B to bf16 copies
                              (round to nearest) and multiply those; outputs stay fp32.
                              Weight gradients and other shapes run the tf32 path.          */
    NNCB_PREC_TF32X3 = 3,  /* fp32-grade tensor-core path ("3xTF32"): every operand v is split
                              into hi = tf32(v) (low 13 mantissa bits cleared) and lo = v - hi,
                              and the contraction runs kind::tf32 over K' = 3K with
                              A' = [A_hi | A_hi | A_lo], B' = [B_hi ; B_lo ; B_hi]
                              (= A_hi B_hi + A_hi B_lo + A_lo B_hi; dropped terms ~2^-21
                              relative). K is concatenated along channels (conv fwd /
                              dgrad, dense) or along the batch (weight gradients).        */
};
enum nncb_epilogue {
    NNCB_EPI_BIAS = 1,
    NNCB_EPI_RELU = 2,
    /* per-output-column sum and sum of squares accumulated (double) into
     * colstats[0:N] / colstats[N:2N] -- BatchNorm statistics fused into the
     * producing GEMM. The GEMM zeroes the accumulator itself.               */
    NNCB_EPI_COLSTATS = 4,
    /* The stored value is the gradient at the input of the ReLU that follows
     * this GEMM's consumer (dgrad epilogue fusion): dy = eg_mask[i] > 0 ?
     * acc (+ eg_res[i]) : 0, eg_mask / eg_res laid out like the output. The
     * BatchNorm backward sums of dy are accumulated alongside (double):
     * eg_sums[0:N] += dy, eg_sums[N:2N] += dy * (eg_x[i] - mean) * invstd with
     * eg_stats = [mean; invstd] (2N floats); the GEMM zeroes eg_sums.
     * Tensor-core path only (returns unhandled otherwise).                   */
    NNCB_EPI_RELU_GRAD = 8,
    /* Hint for NNCB_CONV_WGRAD: the activation `a` holds the same bytes that
     * the most recent NNCB_CONV_FWD on this context read from the same
     * address with the same geometry, and nothing has written it since (in
     * stream order). Lowered copies made by that forward call (the
     * space-to-depth input of a strided small-channel conv) are reused
     * instead of rebuilt. The library re-derives the copy whenever it cannot
     * match the forward call; the caller vouches only for the bytes.       */
    NNCB_EPI_A_UNCHANGED = 16,
    /* Inference BatchNorm of the output column, in the epilogue (forward
     * GEMMs): y = ((acc - bn_mean) * invstd) * bn_gamma + bn_beta with
     * invstd = (float)(1/sqrt((double)bn_var + bn_eps)) per column -- the
     * fused group's NNCB_EW_BN_INFER, operation for operation (bitwise equal
     * to running it as a separate pass); with NNCB_EPI_RELU the ReLU follows. */
    NNCB_EPI_BN_AFFINE = 32,
    /* With NNCB_EPI_BN_AFFINE: residual[row, col] (laid out like the output) is
     * added to the BatchNorm result before the optional ReLU -- an inference
     * residual join, relu(bn(acc) + shortcut), in the epilogue.             */
    NNCB_EPI_RESIDUAL = 64,
};

typedef struct {
    int32_t kind, precision, epilogue;
    /* tensor-core tile choice for this call (a code from nncb_gemm_candidates,
     * e.g. persisted by the layer-wise tuner in the plan); 0 = the table /
     * static rule. A code the shape's route rejects falls back to 0.        */
    int32_t tile;
    /* conv geometry, as kernels::ConvGeom (kernels.hpp:20-25) */
    int64_t n, ih, iw, ci, co, kh, kw, sh, sw, oh, ow, pad_top, pad_left;
    /* dense geometry */
    int64_t batch, in_f, out_f;
    /* NNCB_EPI_COLSTATS accumulator: 2*N doubles */
    double* colstats;
    /* NNCB_EPI_RELU_GRAD operands (see above); eg_res may be NULL */
    const float* eg_mask;
    const float* eg_res;
    const float* eg_x;
    const float* eg_stats;
    double* eg_sums;
    /* NNCB_CONV_FWD: optional K-major copy of the weights, [co][kh*kw*ci],
     * kept current by the caller (nncb_transpose_batch). Tiles that read
     * K-major weights use it instead of transposing per call; routes that
     * lower the weights themselves (space-to-depth, im2col) ignore it.     */
    const float* b_kmajor;
    /* NNCB_EPI_BN_AFFINE operands: per output column (C floats each)        */
    const float* bn_mean;
    const float* bn_var;
    const float* bn_gamma;
    const float* bn_beta;
    double bn_eps;
    /* NNCB_EPI_RESIDUAL operand                                              */
    const float* residual;
    /* Weight gradients (NNCB_CONV_WGRAD / NNCB_DENSE_WGRAD) with sgd_w set:
     * the SGD update of those weights from the gradient this call writes,
     * w = (float)((double)w - (*sgd_lr) * sgd_scale * (double)dW) (reference
     * runtime.cpp:485-496), fused into the split-K fold that produces dW (or
     * issued by the call right after it on the other routes). Valid when no
     * later launch reads the old weights.                                    */
    float* sgd_w;
    const double* sgd_lr;
    double sgd_scale;
    /* With NNCB_EPI_COLSTATS and colstats_finalize set: the call also writes
     * the BatchNorm statistics of its output, colstats_finalize[0:N] = mean,
     * [N:2N] = 1/sqrt(biased var + colstats_eps), exactly as nncb_bn_finalize
     * computes them from the column sums (the finalize launch folded in).   */
    float* colstats_finalize;
    double colstats_eps;
} nncb_gemm_desc;

/* One launch transposing many row-major [rows][cols] matrices into [cols][rows]
 * (e.g. every forward conv's weights into their K-major copies). `jobs` is a
 * device array; tile0 is the exclusive prefix sum of each job's 32x32 tiles,
 * total_tiles the sum.                                                       */
typedef struct {
    const float* src;
    float* dst;
    int32_t rows, cols;
    int64_t tile0;
} nncb_transpose_job;
int nncb_transpose_batch(nncb_ctx* ctx, const nncb_transpose_job* jobs, int n, int64_t total_tiles);

/* float32 sums[0:C] -> out0, sums[C:2C] -> out1 (finalize of NNCB_EPI_RELU_GRAD sums). */
int nncb_colsums_to_float(nncb_ctx* ctx, const double* sums, float* out0, float* out1, int64_t C);

/* FWD:   a = x, b = weight, out = y (bias optional)
 * DGRAD: a = g, b = weight, out = gx
 * WGRAD: a = x, b = g,      out = gw                                    */
/* 1 if the calling thread's last nncb_gemm ran on the tcgen05 tensor-core path, 0 if on the exact fp32 path. */
int nncb_gemm_last_path(void);
/* Route for convolutions with channels % 32 != 0: 1 = builder-warp gather, 0 = im2col (default). */
int nncb_gemm_set_manual_a(int on);
/* Forces the tcgen05 tile: N width (64/128/256) | (1 << 16) for CTA pairs (cta_group::2); 0 = autotune. */
int nncb_gemm_force_tile(int code);
/* GEMM tile choices per shape (they fix the fp32 accumulation order). By
 * default the choice is deterministic: the committed per-shape table
 * (kernels/tile_table.inc, tools/tune_tiles.py) plus imported entries, else a
 * static rule; NNCB_TC_AUTOTUNE=live measures unknown shapes on first use
 * (on a scratch output). Export/import one "key choice" line per shape, so a
 * tuned deployment can persist and reload its choices. Mode: 0 static,
 * 1 table (default), 2 live.                                                */
int nncb_gemm_tuning_export(char* buf, size_t cap, size_t* needed);
int nncb_gemm_tuning_import(const char* text);
int nncb_gemm_tuning_mode(void);
/* Layer-wise tuning support (backends::tune_with_report): the tensor-core tile
 * codes worth timing for this contraction (*n set; codes written up to cap;
 * 0 candidates when the shape has no tensor-core route), and the median
 * device time of `trials` calls with tile `code` after `warmup` calls (CUDA
 * events on the compute stream; `out` is overwritten).                    */
int nncb_gemm_candidates(const nncb_gemm_desc* d, int32_t* codes, int cap, int* n);
int nncb_gemm_time_tile(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b,
                        const float* bias, float* out, int32_t code, int warmup, int trials,
                        float* median_ms);
int nncb_gemm(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b,
              const float* bias, float* out);

/* ------------------------------------------------------------------ */
/*  Pooling (kernels.hpp:258-344)                                       */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t n, ih, iw, c, kh, kw, sh, sw, oh, ow;
} nncb_pool_geom;
/* idx may be NULL; stored as float window-linear index (kernels.hpp:256-283) */
int nncb_maxpool_fwd(nncb_ctx* ctx, const nncb_pool_geom* g, const float* x, float* y,
                     float* idx);
int nncb_maxpool_bwd(nncb_ctx* ctx, const nncb_pool_geom* g, const float* idx, const float* gy,
                     float* gx);
int nncb_avgpool_fwd(nncb_ctx* ctx, int64_t n, int64_t ih, int64_t iw, int64_t c, int64_t oh,
                     int64_t ow, const float* x, float* y);
int nncb_avgpool_bwd(nncb_ctx* ctx, int64_t n, int64_t ih, int64_t iw, int64_t c, int64_t oh,
                     int64_t ow, const float* gy, float* gx);

/* ------------------------------------------------------------------ */
/*  Reductions                                                          */
/* ------------------------------------------------------------------ */
/* out[c] = sum_r x[r, c]  (SumCols kernels.hpp:153-160, SumNHW 245-250).
 * exact = 1: float running sum in row order, bit-identical to the reference;
 * exact = 0: double accumulation in a fixed two-level tree (fast path).      */
int nncb_sum_rows(nncb_ctx* ctx, const float* x, float* out, int64_t rows, int64_t cols, int exact);
/* cumsum along an axis (kernels.hpp:76-111) */
int nncb_cumsum(nncb_ctx* ctx, const float* x, float* y, int64_t outer, int64_t len,
                int64_t inner, int exclusive, int reverse);

/* BatchNorm statistics over rows of x[rows, C]: stats[0:C] = mean, stats[C:2C]
 * = 1/sqrt(var + eps) (biased variance); accumulation in double.           */
int nncb_bn_stats(nncb_ctx* ctx, const float* x, float* stats, int64_t rows, int64_t C,
                  double eps);
/* stats = (mean, 1/sqrt(var + eps)) from fused column sums (NNCB_EPI_COLSTATS). */
int nncb_bn_finalize(nncb_ctx* ctx, const double* colstats, float* stats, int64_t rows, int64_t C, double eps);
/* BatchNorm backward reductions: sum_g[c] = sum g, sum_gx[c] = sum g*xhat.  */
int nncb_bn_grad_reduce(nncb_ctx* ctx, const float* x, const float* stats, const float* g,
                        float* sum_g, float* sum_gx, int64_t rows, int64_t C);
/* LayerNorm over the last axis; gamma/beta [C]; y = xhat*gamma + beta.     */
int nncb_layernorm_fwd(nncb_ctx* ctx, const float* x, const float* gamma, const float* beta,
                       float* y, int64_t rows, int64_t C, double eps);
int nncb_layernorm_bwd(nncb_ctx* ctx, const float* x, const float* gamma, const float* g,
                       float* gx, int64_t rows, int64_t C, double eps);
/* dgamma[c] = sum_r g*xhat (row statistics recomputed)                     */
int nncb_layernorm_dgamma(nncb_ctx* ctx, const float* x, const float* g, float* dgamma,
                          int64_t rows, int64_t C, double eps);
/* LayerNorm backward with the parameter gradients in the same pass:
 * gx as nncb_layernorm_bwd, dgamma[c] = sum_r g*xhat, dbeta[c] = sum_r g
 * (either may be NULL; deterministic per-CTA partials folded in order).   */
int nncb_layernorm_bwd_params(nncb_ctx* ctx, const float* x, const float* gamma, const float* g,
                              float* gx, float* dgamma, float* dbeta, int64_t rows, int64_t C,
                              double eps);

/* ------------------------------------------------------------------ */
/*  Loss and update (runtime.cpp:468-496)                              */
/* ------------------------------------------------------------------ */
/* grad = sign(p - t)/N (sign(0)=0), *loss_dev (double, device) = sum|p-t|/N */
int nncb_l1_loss(nncb_ctx* ctx, const float* pred, const float* target, float* grad,
                 double* loss_dev, int64_t n);
/* Softmax cross-entropy over the last axis of logits [rows, C] with
 * probability-vector targets (extension loss; the reference has only L1):
 * *loss_dev = -(1/rows) sum_r sum_c t log softmax(z)_c, computed in double;
 * grad = (softmax(z) - t)/rows. Deterministic (fixed reduction order).     */
int nncb_softmax_ce(nncb_ctx* ctx, const float* logits, const float* target, float* grad, double* loss_dev,
                    int64_t rows, int64_t C);
/* Flat-buffer SGD over the whole parameter region (weights and gradients share
 * one layout): w = (float)((double)w - lr*((double)g*grad_scale)). With
 * grad_scale = 1 this is bit-identical to runtime::sgd_step (runtime.cpp:493). */
int nncb_sgd(nncb_ctx* ctx, float* w, const float* g, int64_t n, double lr, double grad_scale);
/* The same update with the learning rate read from device memory (*lr_dev),
 * launched on context stream `stream` (a bucket's update on the comm stream
 * right after its all-reduce, overlapping the rest of the backward pass).  */
int nncb_sgd_dev(nncb_ctx* ctx, int stream, float* w, const float* g, int64_t n, const double* lr_dev,
                 double grad_scale);
/* The same update over n_ranges element ranges of w / g in one launch:
 * ranges_dev = device [offset0, count0, offset1, count1, ...] (int64,
 * offsets 16-byte aligned); max_count sizes the grid.                      */
int nncb_sgd_dev_ranges(nncb_ctx* ctx, int stream, float* w, const float* g, const int64_t* ranges_dev,
                        int n_ranges, int64_t max_count, const double* lr_dev, double grad_scale);

/* ------------------------------------------------------------------ */
/*  Data-parallel collectives (NCCL over NVLink/NVSwitch)               */
/* ------------------------------------------------------------------ */
int nncb_comm_unique_id(uint8_t id[128]);
int nncb_comm_init(nncb_ctx* ctx, int nranks, int rank, const uint8_t id[128]);
int nncb_comm_destroy(nncb_ctx* ctx);
/* in-place sum all-reduce of fp32 on the comm stream, ordered after all work
 * enqueued so far on the compute stream; the compute stream waits for it.  */
int nncb_allreduce_sum(nncb_ctx* ctx, float* buf, int64_t count);
/* Overlapped variant: the comm stream waits for the compute stream's current
 * position and all-reduces there; the compute stream continues without
 * waiting. nncb_comm_join makes the compute stream wait for every collective
 * issued so far (before the buffers are read, e.g. by SGD).                 */
int nncb_allreduce_sum_async(nncb_ctx* ctx, float* buf, int64_t count);
int nncb_comm_join(nncb_ctx* ctx);
/* The all-reduce alone, on the comm stream (the caller forks/joins).       */
int nncb_allreduce_sum_on_comm(nncb_ctx* ctx, float* buf, int64_t count);
/* 1 if a communicator is initialised on this context.                      */
int nncb_comm_active(nncb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NNCB_H */
