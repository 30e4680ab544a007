// gemm_simt.cu -- exact-order fp32 implicit GEMM (NNCB_PREC_FP32, parity mode).
//
// All six contractions of the reference (kernels.hpp:118-243) as one tiled
// implicit GEMM C[M,N] = sum_k A[m,k] B[k,n] whose per-output accumulation
// visits k in exactly the reference loop order with separately rounded
// products (__fmul_rn/__fadd_rn, no FMA), so results are bit-identical to the
// reference REF / GEMM_TILED CPU kernels:
//   dense fwd    acc = bias; k = i ascending                 (kernels.hpp:118-127)
//   dense dgrad  acc = 0;    k = o ascending                 (kernels.hpp:130-139)
//   dense wgrad  acc = 0;    k = b ascending                 (kernels.hpp:142-151)
//   conv fwd     acc = bias; k = (dh, dw, ci) ascending      (kernels.hpp:166-190)
//   conv wgrad   acc = 0;    k = (n, oh, ow) ascending       (kernels.hpp:220-243)
//   conv dgrad   acc = 0;    per tap (oh, ow) ascending == (dh, dw) descending, an
//                inner sum over co is rounded before it is added (kernels.hpp:192-218)
// Out-of-range taps contribute exact zeros. The tensor-core path (gemm_tc.cu)
// is the production path; this kernel pins it and serves the fp32 mode.
#include "nncb_internal.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

struct Geo {
    int64_t M, N, K;
    nncb_gemm_desc d;
};

template <int KIND>
__device__ __forceinline__ float a_val(const float* __restrict__ a, const Geo& G, int64_t m, int64_t k) {
    const nncb_gemm_desc& d = G.d;
    if (m >= G.M || k >= G.K) return 0.f;
    if (KIND == NNCB_DENSE_FWD) return a[m * d.in_f + k];
    if (KIND == NNCB_DENSE_DGRAD) return a[m * d.out_f + k];
    if (KIND == NNCB_DENSE_WGRAD) return a[k * d.in_f + m];
    if (KIND == NNCB_CONV_FWD) {
        int64_t ci = k % d.ci, t = k / d.ci, dw = t % d.kw, dh = t / d.kw;
        int64_t ow = m % d.ow, r = m / d.ow, oh = r % d.oh, n = r / d.oh;
        int64_t h = oh * d.sh + dh - d.pad_top, w = ow * d.sw + dw - d.pad_left;
        if (h < 0 || h >= d.ih || w < 0 || w >= d.iw) return 0.f;
        return a[((n * d.ih + h) * d.iw + w) * d.ci + ci];
    }
    if (KIND == NNCB_CONV_WGRAD) {  // m = (dh, dw, ci), k = (n, oh, ow)
        int64_t ci = m % d.ci, t = m / d.ci, dw = t % d.kw, dh = t / d.kw;
        int64_t ow = k % d.ow, r = k / d.ow, oh = r % d.oh, n = r / d.oh;
        int64_t h = oh * d.sh + dh - d.pad_top, w = ow * d.sw + dw - d.pad_left;
        if (h < 0 || h >= d.ih || w < 0 || w >= d.iw) return 0.f;
        return a[((n * d.ih + h) * d.iw + w) * d.ci + ci];
    }
    return 0.f;
}

template <int KIND>
__device__ __forceinline__ float b_val(const float* __restrict__ b, const Geo& G, int64_t k, int64_t n) {
    const nncb_gemm_desc& d = G.d;
    if (k >= G.K || n >= G.N) return 0.f;
    if (KIND == NNCB_DENSE_FWD) return b[k * d.out_f + n];
    if (KIND == NNCB_DENSE_DGRAD) return b[n * d.out_f + k];
    if (KIND == NNCB_DENSE_WGRAD) return b[k * d.out_f + n];
    if (KIND == NNCB_CONV_FWD) return b[k * d.co + n];
    if (KIND == NNCB_CONV_WGRAD) return b[k * d.co + n];
    return 0.f;
}

template <int KIND>
__global__ void __launch_bounds__(256) gemm_exact_k(const float* __restrict__ a, const float* __restrict__ b,
                                                   const float* __restrict__ bias, float* __restrict__ out, Geo G) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t n = n0 + tx * 4 + j;
            acc[i][j] = (bias && n < G.N) ? bias[n] : 0.f;
        }
    for (int64_t k0 = 0; k0 < G.K; k0 += BK) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int idx = threadIdx.x + e * 256;
            int kk = idx % BK, mm = idx / BK;
            As[kk][mm] = a_val<KIND>(a, G, m0 + mm, k0 + kk);
            int nn = idx % BN, kb = idx / BN;
            Bs[kb][nn] = b_val<KIND>(b, G, k0 + kb, n0 + nn);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            if (k0 + kk >= G.K) break;
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int64_t m = m0 + ty * 4 + i;
        if (m >= G.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t n = n0 + tx * 4 + j;
            if (n < G.N) out[m * G.N + n] = acc[i][j];
        }
    }
}

// Conv dgrad with the reference's two-level rounding: for output pixel m=(n,h,w)
// and channel ci, taps are visited in (dh, dw) DESCENDING order (== (oh, ow)
// ascending); each valid tap contributes its own rounded sum over co.
__global__ void __launch_bounds__(256) conv_dgrad_exact_k(const float* __restrict__ g, const float* __restrict__ k,
                                                         float* __restrict__ gx, Geo G) {
    const nncb_gemm_desc& d = G.d;
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    float acc[4][4] = {};
    for (int64_t tap = d.kh * d.kw - 1; tap >= 0; --tap) {
        const int64_t dh = tap / d.kw, dw = tap % d.kw;
        float part[4][4] = {};
        for (int64_t c0 = 0; c0 < d.co; c0 += BK) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int idx = threadIdx.x + e * 256;
                int kk = idx % BK, mm = idx / BK;
                int64_t m = m0 + mm, co = c0 + kk;
                float v = 0.f;
                if (m < G.M && co < d.co) {
                    int64_t w = m % d.iw, r = m / d.iw, h = r % d.ih, n = r / d.ih;
                    int64_t th = h + d.pad_top - dh, tw = w + d.pad_left - dw;
                    if (th >= 0 && tw >= 0 && th % d.sh == 0 && tw % d.sw == 0) {
                        int64_t oh = th / d.sh, ow = tw / d.sw;
                        if (oh < d.oh && ow < d.ow) v = g[((n * d.oh + oh) * d.ow + ow) * d.co + co];
                    }
                }
                As[kk][mm] = v;
                int nn = idx % BN, kb = idx / BN;
                int64_t ci = n0 + nn, cob = c0 + kb;
                Bs[kb][nn] = (ci < d.ci && cob < d.co) ? k[((dh * d.kw + dw) * d.ci + ci) * d.co + cob] : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                if (c0 + kk >= d.co) break;
                float av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) part[i][j] = __fadd_rn(part[i][j], __fmul_rn(av[i], bv[j]));
            }
            __syncthreads();
        }
        // add this tap's rounded partial only where the tap is valid for the row
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int64_t m = m0 + ty * 4 + i;
            bool valid = false;
            if (m < G.M) {
                int64_t w = m % d.iw, r = m / d.iw, h = r % d.ih;
                int64_t th = h + d.pad_top - dh, tw = w + d.pad_left - dw;
                valid = th >= 0 && tw >= 0 && th % d.sh == 0 && tw % d.sw == 0 && th / d.sh < d.oh && tw / d.sw < d.ow;
            }
            if (valid)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], part[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int64_t m = m0 + ty * 4 + i;
        if (m >= G.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t n = n0 + tx * 4 + j;
            if (n < G.N) gx[m * G.N + n] = acc[i][j];
        }
    }
}

}  // namespace

namespace nncb {

int gemm_simt(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias, float* out) {
    Geo G{};
    G.d = *d;
    switch (d->kind) {
        case NNCB_DENSE_FWD: G.M = d->batch; G.N = d->out_f; G.K = d->in_f; break;
        case NNCB_DENSE_DGRAD: G.M = d->batch; G.N = d->in_f; G.K = d->out_f; break;
        case NNCB_DENSE_WGRAD: G.M = d->in_f; G.N = d->out_f; G.K = d->batch; break;
        case NNCB_CONV_FWD: G.M = d->n * d->oh * d->ow; G.N = d->co; G.K = d->kh * d->kw * d->ci; break;
        case NNCB_CONV_WGRAD: G.M = d->kh * d->kw * d->ci; G.N = d->co; G.K = d->n * d->oh * d->ow; break;
        case NNCB_CONV_DGRAD: G.M = d->n * d->ih * d->iw; G.N = d->ci; G.K = d->kh * d->kw * d->co; break;
        default: return fail("gemm: unknown kind");
    }
    if (G.M == 0 || G.N == 0) return 0;
    if ((G.N + BN - 1) / BN > 0x7fffffff || (G.M + BM - 1) / BM > 65535 * 1024)
        return fail("gemm: problem too large for the exact path");
    dim3 grid((unsigned)((G.N + BN - 1) / BN), (unsigned)((G.M + BM - 1) / BM));
    if (grid.y > 65535) return fail("gemm exact: M too large (grid.y > 65535); use the tensor-core path");
    const float* bi = (d->epilogue & NNCB_EPI_BIAS) ? bias : nullptr;
    switch (d->kind) {
        case NNCB_DENSE_FWD: gemm_exact_k<NNCB_DENSE_FWD><<<grid, 256, 0, ctx->stream>>>(a, b, bi, out, G); break;
        case NNCB_DENSE_DGRAD: gemm_exact_k<NNCB_DENSE_DGRAD><<<grid, 256, 0, ctx->stream>>>(a, b, nullptr, out, G); break;
        case NNCB_DENSE_WGRAD: gemm_exact_k<NNCB_DENSE_WGRAD><<<grid, 256, 0, ctx->stream>>>(a, b, nullptr, out, G); break;
        case NNCB_CONV_FWD: gemm_exact_k<NNCB_CONV_FWD><<<grid, 256, 0, ctx->stream>>>(a, b, bi, out, G); break;
        case NNCB_CONV_WGRAD: gemm_exact_k<NNCB_CONV_WGRAD><<<grid, 256, 0, ctx->stream>>>(a, b, nullptr, out, G); break;
        case NNCB_CONV_DGRAD: conv_dgrad_exact_k<<<grid, 256, 0, ctx->stream>>>(a, b, out, G); break;
    }
    NNCB_LAUNCHED(ctx);
    return 0;
}

}  // namespace nncb

namespace {
thread_local int g_last_path = -1;
}

// Which kernel family ran the calling thread's last nncb_gemm: 1 = tcgen05
// (tf32 tensor cores), 0 = exact fp32 path. Lets tests prove the path taken.
extern "C" int nncb_gemm_last_path(void) { return g_last_path; }

namespace {
__global__ void affine_relu_k(float* __restrict__ y, const float* __restrict__ mean, const float* __restrict__ var,
                              const float* __restrict__ gamma, const float* __restrict__ beta,
                              const float* __restrict__ res, int64_t rows, int64_t C, double eps, int relu) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * C; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % C;
        const float inv = static_cast<float>(1.0 / sqrt(static_cast<double>(var[c]) + eps));
        float v = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(y[i], mean[c]), inv), gamma[c]), beta[c]);
        if (res) v = __fadd_rn(v, res[i]);
        if (relu) v = v > 0.f ? v : 0.f;
        y[i] = v;
    }
}
}  // namespace

namespace nncb {
int affine_relu_output(nncb_ctx* ctx, const nncb_gemm_desc* d, float* out) {
    const bool dense = d->kind == NNCB_DENSE_FWD;
    if (d->kind != NNCB_DENSE_FWD && d->kind != NNCB_CONV_FWD) return fail("BN_AFFINE is a forward-GEMM epilogue");
    const int64_t rows = dense ? d->batch : d->n * d->oh * d->ow, C = dense ? d->out_f : d->co;
    affine_relu_k<<<grid_for(ctx, rows * C, 256), 256, 0, ctx->stream>>>(out, d->bn_mean, d->bn_var, d->bn_gamma,
                                                                        d->bn_beta,
                                                                        (d->epilogue & NNCB_EPI_RESIDUAL) ? d->residual : nullptr,
                                                                        rows, C, d->bn_eps,
                                                                        (d->epilogue & NNCB_EPI_RELU) ? 1 : 0);
    NNCB_LAUNCHED(ctx);
    return 0;
}
}  // namespace nncb

int nncb_gemm_core(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
                   float* out);

// Weight gradients with sgd_w: the update is fused into the split-K fold when
// the tensor-core route produced dW that way, else applied right after.
extern "C" int nncb_gemm(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
                         float* out) {
    nncb::take_sgd_applied();
    const int rc = nncb_gemm_core(ctx, d, a, b, bias, out);
    const bool fused = nncb::take_sgd_applied();
    if (rc || !d->sgd_w || fused) return rc;
    if (d->kind != NNCB_CONV_WGRAD && d->kind != NNCB_DENSE_WGRAD) return 0;
    if (!d->sgd_lr) return nncb::fail("nncb_gemm: sgd_w needs sgd_lr");
    const int64_t count = d->kind == NNCB_DENSE_WGRAD ? d->in_f * d->out_f : d->kh * d->kw * d->ci * d->co;
    return nncb_sgd_dev(ctx, NNCB_STREAM_COMPUTE, d->sgd_w, out, count, d->sgd_lr, d->sgd_scale);
}

int nncb_gemm_core(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
                   float* out) {
    const bool colstats = (d->epilogue & NNCB_EPI_COLSTATS) && d->colstats;
    if (colstats && d->kind != NNCB_CONV_FWD && d->kind != NNCB_DENSE_FWD)
        return nncb::fail("nncb_gemm: column statistics are a forward-GEMM epilogue");
    if (d->precision == NNCB_PREC_TF32 || d->precision == NNCB_PREC_BF16) {
        bool handled = false;
        int rc = nncb::gemm_tc(ctx, d, a, b, bias, out, &handled);
        g_last_path = 1;
        if (rc || handled) return rc;
    } else if (d->precision == NNCB_PREC_TF32X3) {
        bool handled = false;
        int rc = nncb::gemm_tc_x3(ctx, d, a, b, bias, out, &handled);
        g_last_path = 1;
        if (rc || handled) return rc;
    }
    if (d->epilogue & NNCB_EPI_RELU_GRAD)
        return nncb::fail("nncb_gemm: NNCB_EPI_RELU_GRAD is a tensor-core epilogue (tf32 precision, TMA-eligible shape)");
    g_last_path = 0;
    if (int rc = nncb::gemm_simt(ctx, d, a, b, bias, out)) return rc;
    if (d->epilogue & NNCB_EPI_BN_AFFINE)   // the exact path applies the epilogue as a pass over its output
        if (int rc = nncb::affine_relu_output(ctx, d, out)) return rc;
    if (colstats) {
        const bool dense = d->kind == NNCB_DENSE_FWD;
        const int64_t rows = dense ? d->batch : d->n * d->oh * d->ow, C = dense ? d->out_f : d->co;
        if (int rc = nncb::colstats_from_output(ctx, out, d->colstats, rows, C)) return rc;
        if (d->colstats_finalize) return nncb_bn_finalize(ctx, d->colstats, d->colstats_finalize, rows, C, d->colstats_eps);
        return 0;
    }
    return 0;
}
