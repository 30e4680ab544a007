// fused_ops.cu -- the non-GEMM members of fused groups: pooling, reductions,
// BatchNorm / LayerNorm statistics, L1 loss and the SGD update.
//
// Bit-exactness notes (vs the reference CPU kernels):
//  * maxpool fwd: strict '>' scan in window order, first max wins, index stored
//    as float (kernels.hpp:258-284) -> bit-exact.
//  * maxpool bwd / avgpool bwd are written as GATHERS (no atomics): each input
//    element sums its contributions in increasing (oh, ow) order starting from
//    +0, exactly the order the reference's scatter-add loop (kernels.hpp:286-344)
//    applies them -> bit-exact.
//  * avgpool fwd accumulates the window in (h, w) order then multiplies by
//    T(1)/T(count) (kernels.hpp:304-322) -> bit-exact.
//  * cumsum is sequential along the axis per line (kernels.hpp:76-111) -> bit-exact.
//  * column sums (SumCols/SumNHW), BN/LN statistics accumulate in double with a
//    fixed (deterministic) two-level order: more accurate than the reference's
//    float running sum; compared against the oracle with a tolerance.
//  * L1 gradient and SGD are computed in double per element and cast, exactly
//    like runtime.cpp:468-496 -> bit-exact; the loss is a double tree sum.
#include <algorithm>

#include "nncb_internal.cuh"

namespace {

// Max pooling, 4 channels per thread (C % 4 == 0: float4 loads/stores) or 1.
// Pixel decomposition in 32-bit (host guarantees n*oh*ow < 2^31).
template <int V>
__global__ void maxpool_fwd_k(const float* __restrict__ x, float* __restrict__ y, float* __restrict__ idx,
                              nncb_pool_geom g) {
    const int C = (int)g.c, CV = C / V;
    const int OW = (int)g.ow, OH = (int)g.oh, IW = (int)g.iw, IH = (int)g.ih;
    const int64_t total = g.n * g.oh * g.ow * CV;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int cv = (int)(t % CV);
        const int64_t pix = t / CV;
        const int ow = (int)(pix % OW);
        const int64_t r = pix / OW;
        const int oh = (int)(r % OH);
        const int64_t n = r / OH;
        float best[V];
        int bi[V];
#pragma unroll
        for (int j = 0; j < V; ++j) bi[j] = -1;
        const float* base = x + (n * IH * (int64_t)IW) * C + cv * V;
        for (int dh = 0; dh < (int)g.kh; ++dh)
            for (int dw = 0; dw < (int)g.kw; ++dw) {
                const int h = oh * (int)g.sh + dh, w = ow * (int)g.sw + dw;
                const float* p = base + ((int64_t)h * IW + w) * C;
                float v[V];
                if (V == 4) {
                    float4 q = __ldg(reinterpret_cast<const float4*>(p));
                    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
                } else {
                    v[0] = __ldg(p);
                }
                const int k = dh * (int)g.kw + dw;
#pragma unroll
                for (int j = 0; j < V; ++j)
                    if (bi[j] < 0 || v[j] > best[j]) {
                        best[j] = v[j];
                        bi[j] = k;
                    }
            }
        const int64_t at = pix * C + cv * V;
        if (V == 4) {
            *reinterpret_cast<float4*>(y + at) = make_float4(best[0], best[1], best[2], best[3]);
            if (idx) *reinterpret_cast<float4*>(idx + at) = make_float4((float)bi[0], (float)bi[1], (float)bi[2], (float)bi[3]);
        } else {
            y[at] = best[0];
            if (idx) idx[at] = (float)bi[0];
        }
    }
}

// Max-pool backward as a gather over the windows covering each input pixel,
// in (oh, ow) ascending order = the reference scatter order (bit-exact).
// K3S2 = 1: the 3x3 stride-2 window (ResNet stem) with compile-time window
// arithmetic; 0: window and stride from the descriptor.
template <int V, typename I, int K3S2 = 0>
__global__ void maxpool_bwd_k(const float* __restrict__ idx, const float* __restrict__ gy, float* __restrict__ gx,
                              nncb_pool_geom g) {
    const int C = (int)g.c, CV = C / V;
    const int OW = (int)g.ow, OH = (int)g.oh, IW = (int)g.iw, IH = (int)g.ih;
    const int KH = K3S2 ? 3 : (int)g.kh, KW = K3S2 ? 3 : (int)g.kw, SH = K3S2 ? 2 : (int)g.sh, SW = K3S2 ? 2 : (int)g.sw;
    const I total = static_cast<I>(g.n * g.ih * g.iw * CV);
    for (I t = blockIdx.x * (I)blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
        const int cv = (int)(t % CV);
        const I pix = t / CV;
        const int w = (int)(pix % IW);
        const I r = pix / IW;
        const int h = (int)(r % IH);
        const I n = r / IH;
        const int oh0 = h - KH + 1 > 0 ? (h - KH + SH) / SH : 0;
        const int oh1 = min(h / SH, OH - 1);
        const int ow0 = w - KW + 1 > 0 ? (w - KW + SW) / SW : 0;
        const int ow1 = min(w / SW, OW - 1);
        float acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = 0.f;
        for (int oh = oh0; oh <= oh1; ++oh)
            for (int ow = ow0; ow <= ow1; ++ow) {
                const int want = (h - oh * SH) * KW + (w - ow * SW);
                const I at = ((n * OH + oh) * OW + ow) * C + cv * V;
                if (V == 4) {
                    float4 ix = __ldg(reinterpret_cast<const float4*>(idx + at));
                    float4 gv = __ldg(reinterpret_cast<const float4*>(gy + at));
                    if ((int)ix.x == want) acc[0] = __fadd_rn(acc[0], gv.x);
                    if ((int)ix.y == want) acc[1] = __fadd_rn(acc[1], gv.y);
                    if ((int)ix.z == want) acc[2] = __fadd_rn(acc[2], gv.z);
                    if ((int)ix.w == want) acc[3] = __fadd_rn(acc[3], gv.w);
                } else {
                    if ((int)__ldg(idx + at) == want) acc[0] = __fadd_rn(acc[0], __ldg(gy + at));
                }
            }
        const I o = pix * C + cv * V;
        if (V == 4)
            *reinterpret_cast<float4*>(gx + o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        else
            gx[o] = acc[0];
    }
}

// 3x3 stride-2 max pooling (the ResNet stem), 4 channels per thread, 32-bit
// index decode (host: element counts < 2^31). All nine window rows are loaded
// before the compare chain, which keeps the reference's scan order.
__global__ void maxpool_fwd_k33(const float* __restrict__ x, float* __restrict__ y, float* __restrict__ idx,
                                nncb_pool_geom g) {
    const uint32_t C = (uint32_t)g.c, CV = C / 4, OW = (uint32_t)g.ow, OH = (uint32_t)g.oh;
    const uint32_t IW = (uint32_t)g.iw, IH = (uint32_t)g.ih;
    const uint32_t total = (uint32_t)(g.n * g.oh * g.ow) * CV;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const uint32_t pix = t / CV, cv = t - pix * CV;
        const uint32_t r = pix / OW, ow = pix - r * OW;
        const uint32_t n = r / OH, oh = r - n * OH;
        const float* p0 = x + ((size_t)(n * IH + 2 * oh) * IW + 2 * ow) * C + cv * 4;
        float4 v[9];
#pragma unroll
        for (int dh = 0; dh < 3; ++dh)
#pragma unroll
            for (int dw = 0; dw < 3; ++dw) v[dh * 3 + dw] = __ldg(reinterpret_cast<const float4*>(p0 + ((size_t)dh * IW + dw) * C));
        float4 best = v[0];
        float4 bi = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 1; k < 9; ++k) {   // strict '>': the first maximum in window order wins
            if (v[k].x > best.x) { best.x = v[k].x; bi.x = (float)k; }
            if (v[k].y > best.y) { best.y = v[k].y; bi.y = (float)k; }
            if (v[k].z > best.z) { best.z = v[k].z; bi.z = (float)k; }
            if (v[k].w > best.w) { best.w = v[k].w; bi.w = (float)k; }
        }
        const size_t at = (size_t)pix * C + cv * 4;
        *reinterpret_cast<float4*>(y + at) = best;
        if (idx) *reinterpret_cast<float4*>(idx + at) = bi;
    }
}

// 3x3 stride-2 max-pool backward over 2x2 input blocks: rows 2a, 2a+1 and
// columns 2b, 2b+1 are covered only by windows oh in {a-1, a}, ow in {b-1, b}
// (odd rows / columns by a / b alone). Each thread loads those four windows
// once (index and gradient) and writes its block, every pixel adding its
// windows in ascending (oh, ow) order -- the reference's scatter order.
__global__ void maxpool_bwd_k33(const float* __restrict__ idx, const float* __restrict__ gy, float* __restrict__ gx,
                                nncb_pool_geom g) {
    const uint32_t C = (uint32_t)g.c, CV = C / 4, OW = (uint32_t)g.ow, OH = (uint32_t)g.oh;
    const uint32_t IW = (uint32_t)g.iw, IH = (uint32_t)g.ih, BW = (IW + 1) / 2, BH = (IH + 1) / 2;
    const uint32_t total = (uint32_t)g.n * BH * BW * CV;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const uint32_t blk = t / CV, cv = t - blk * CV;
        const uint32_t r = blk / BW, b = blk - r * BW;
        const uint32_t n = r / BH, a = r - n * BH;
        // windows q = (a-1, b-1), (a-1, b), (a, b-1), (a, b)
        float4 ix[4], gv[4];
        bool on[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int oh = (int)a - 1 + (q >> 1), ow = (int)b - 1 + (q & 1);
            on[q] = oh >= 0 && oh < (int)OH && ow >= 0 && ow < (int)OW;
            const size_t at = on[q] ? ((size_t)(n * OH + oh) * OW + ow) * C + cv * 4 : 0;
            ix[q] = on[q] ? __ldg(reinterpret_cast<const float4*>(idx + at)) : make_float4(-1.f, -1.f, -1.f, -1.f);
            gv[q] = on[q] ? __ldg(reinterpret_cast<const float4*>(gy + at)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                const uint32_t h = 2 * a + dy, w = 2 * b + dx;
                if (h >= IH || w >= IW) continue;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int wy = q >> 1, wx = q & 1;   // window row a-1+wy, column b-1+wx
                    if ((dy == 1 && wy == 0) || (dx == 1 && wx == 0)) continue;   // odd rows/cols: one window
                    // offset of pixel (h, w) inside window (a-1+wy, b-1+wx)
                    const float want = (float)((dy + 2 * (1 - wy)) * 3 + (dx + 2 * (1 - wx)));
                    if (!on[q]) continue;
                    if (ix[q].x == want) acc[0] = __fadd_rn(acc[0], gv[q].x);
                    if (ix[q].y == want) acc[1] = __fadd_rn(acc[1], gv[q].y);
                    if (ix[q].z == want) acc[2] = __fadd_rn(acc[2], gv[q].z);
                    if (ix[q].w == want) acc[3] = __fadd_rn(acc[3], gv[q].w);
                }
                *reinterpret_cast<float4*>(gx + ((size_t)(n * IH + h) * IW + w) * C + cv * 4) =
                    make_float4(acc[0], acc[1], acc[2], acc[3]);
            }
    }
}

__device__ __forceinline__ int64_t a_start(int64_t o, int64_t in, int64_t out) { return (o * in) / out; }
__device__ __forceinline__ int64_t a_end(int64_t o, int64_t in, int64_t out) { return ((o + 1) * in + out - 1) / out; }

__global__ void avgpool_fwd_k(const float* __restrict__ x, float* __restrict__ y, int64_t n, int64_t ih, int64_t iw,
                              int64_t c, int64_t oh, int64_t ow) {
    int64_t total = n * oh * ow * c;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t ch = t % c;
        int64_t r = t / c;
        int64_t p = r % ow;
        r /= ow;
        int64_t o = r % oh;
        int64_t b = r / oh;
        int64_t h0 = a_start(o, ih, oh), h1 = a_end(o, ih, oh), w0 = a_start(p, iw, ow), w1 = a_end(p, iw, ow);
        float scale = __fdiv_rn(1.f, static_cast<float>((h1 - h0) * (w1 - w0)));
        float acc = 0.f;
        for (int64_t h = h0; h < h1; ++h)
            for (int64_t w = w0; w < w1; ++w) acc = __fadd_rn(acc, __ldg(x + ((b * ih + h) * iw + w) * c + ch));
        y[t] = __fmul_rn(acc, scale);
    }
}

// Global average pool (1x1 output), 4 channels per thread, 32-bit indices:
// the window is summed in the same (h, w) order as avgpool_fwd_k (bit-identical)
// but the 4-wide loads are independent, so the pool streams instead of chaining
// 64-bit index math per element.
__global__ void avgpool_fwd_global4_k(const float* __restrict__ x, float* __restrict__ y, uint32_t hw, uint32_t c4,
                                      uint32_t total4, float scale) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total4; t += gridDim.x * blockDim.x) {
        const uint32_t ch4 = t % c4, b = t / c4;
        const float4* src = reinterpret_cast<const float4*>(x) + static_cast<size_t>(b) * hw * c4 + ch4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 7
        for (uint32_t p = 0; p < hw; ++p) {
            const float4 v = __ldg(src + static_cast<size_t>(p) * c4);
            acc.x = __fadd_rn(acc.x, v.x);
            acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z);
            acc.w = __fadd_rn(acc.w, v.w);
        }
        reinterpret_cast<float4*>(y)[t] =
            make_float4(__fmul_rn(acc.x, scale), __fmul_rn(acc.y, scale), __fmul_rn(acc.z, scale), __fmul_rn(acc.w, scale));
    }
}

// Output windows containing input row h: o in [o_lo(h), o_hi(h)] where
// a_start(o) <= h < a_end(o); found by stepping from the proportional guess
// (adaptive windows overlap by at most one position, so the loops run <= 2
// steps). Contributions accumulate in (o, p) ascending order, as the
// reference's output-major scatter does.
__device__ __forceinline__ void a_range(int h, int in, int out, int& lo, int& hi) {
    int o = static_cast<int>((static_cast<int64_t>(h) * out) / in);
    while (o > 0 && a_end(o - 1, in, out) > h) --o;
    while (o < out && a_end(o, in, out) <= h) ++o;
    lo = o;
    int e = o;
    while (e + 1 < out && a_start(e + 1, in, out) <= h) ++e;
    hi = e;
}

// Global average pooling backward (1x1 output): every input element of
// image b, channel c receives 0 + gy[b, c] * (1 / (IH*IW)) -- the general
// kernel's arithmetic for its single window (the +0 keeps a -0 product +0).
__global__ void avgpool_bwd_global_k(const float* __restrict__ gy, float* __restrict__ gx, uint32_t hw, uint32_t CV,
                                     uint32_t total) {
    const float scale = __fdiv_rn(1.f, static_cast<float>(hw));
    const uint32_t per_image = hw * CV;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const uint32_t b = t / per_image, cv = (t - b * per_image) % CV;
        const float4 q = __ldg(reinterpret_cast<const float4*>(gy) + (size_t)b * CV + cv);
        reinterpret_cast<float4*>(gx)[t] =
            make_float4(__fadd_rn(0.f, __fmul_rn(q.x, scale)), __fadd_rn(0.f, __fmul_rn(q.y, scale)),
                        __fadd_rn(0.f, __fmul_rn(q.z, scale)), __fadd_rn(0.f, __fmul_rn(q.w, scale)));
    }
}

template <int V, typename I>
__global__ void avgpool_bwd_k(const float* __restrict__ gy, float* __restrict__ gx, int64_t n, int64_t ih, int64_t iw,
                              int64_t c, int64_t oh, int64_t ow) {
    const int C = (int)c, CV = C / V, IH = (int)ih, IW = (int)iw, OH = (int)oh, OW = (int)ow;
    const I total = static_cast<I>(n * ih * iw * CV);
    for (I t = blockIdx.x * (I)blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
        const int cv = (int)(t % CV);
        I r = t / CV;
        const int w = (int)(r % IW);
        r /= IW;
        const int h = (int)(r % IH);
        const I b = r / IH;
        int o0, o1, p0, p1;
        a_range(h, IH, OH, o0, o1);
        a_range(w, IW, OW, p0, p1);
        float acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = 0.f;
        for (int o = o0; o <= o1; ++o) {
            const int h0 = (int)a_start(o, IH, OH), h1 = (int)a_end(o, IH, OH);
            for (int p = p0; p <= p1; ++p) {
                const int w0 = (int)a_start(p, IW, OW), w1 = (int)a_end(p, IW, OW);
                const float scale = __fdiv_rn(1.f, static_cast<float>((h1 - h0) * (w1 - w0)));
                const float* src = gy + ((b * OH + o) * OW + p) * C + cv * V;
                float v[V];
                if (V == 4) {
                    const float4 q = __ldg(reinterpret_cast<const float4*>(src));
                    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
                } else {
                    v[0] = __ldg(src);
                }
#pragma unroll
                for (int j = 0; j < V; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(v[j], scale));
            }
        }
        float* dst = gx + t * V;
        if (V == 4)
            *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        else
            dst[0] = acc[0];
    }
}

// Column reductions over x[rows, C]: block (32 x 8) handles a 32-column tile
// and a chunk of rows; partial sums (double) go to part[chunk][C] and a second
// pass folds the chunks in order.
template <int MODE>
__global__ void col_partial_k(const float* __restrict__ x, const float* __restrict__ g, const float* __restrict__ stats,
                              double* __restrict__ part, int64_t rows, int64_t C, int64_t rows_per_chunk) {
    int64_t col = blockIdx.x * 32 + threadIdx.x;
    int64_t chunk = blockIdx.y;
    int64_t r0 = chunk * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
    double s0 = 0, s1 = 0;
    if (col < C) {
        float mean = 0.f, invstd = 0.f;
        if (MODE == 2) {
            mean = stats[col];
            invstd = stats[C + col];
        }
        for (int64_t r = r0 + threadIdx.y; r < r1; r += blockDim.y) {
            float v = __ldg(x + r * C + col);
            if (MODE == 0) {
                s0 += v;
            } else if (MODE == 1) {
                s0 += v;
                s1 += (double)v * (double)v;
            } else {
                float gv = __ldg(g + r * C + col);
                double xhat = ((double)v - (double)mean) * (double)invstd;
                s0 += gv;
                s1 += (double)gv * xhat;
            }
        }
    }
    __shared__ double sh0[8][33], sh1[8][33];
    sh0[threadIdx.y][threadIdx.x] = s0;
    sh1[threadIdx.y][threadIdx.x] = s1;
    __syncthreads();
    if (threadIdx.y == 0 && col < C) {
        for (int k = 1; k < (int)blockDim.y; ++k) {
            s0 += sh0[k][threadIdx.x];
            s1 += sh1[k][threadIdx.x];
        }
        part[(chunk * 2 + 0) * C + col] = s0;
        part[(chunk * 2 + 1) * C + col] = s1;
    }
}

// Vectorised variant for C % 4 == 0: each thread owns float4 channel groups,
// `tpr` threads cover a row, 256 / tpr rows advance per iteration; the partial
// (double) sums of the threads sharing a channel group are folded in smem.
template <int MODE>
__global__ void __launch_bounds__(256) col_partial4_k(const float* __restrict__ x, const float* __restrict__ g,
                                                      const float* __restrict__ stats, double* __restrict__ part,
                                                      int64_t rows, int64_t C, int64_t rows_per_chunk) {
    __shared__ double red[2][256][4];
    const int C4 = (int)(C / 4);
    const int tpr = C4 < 256 ? C4 : 256, rpi = 256 / tpr;
    const int lt = threadIdx.x % tpr, rr = threadIdx.x / tpr;
    const int64_t chunk = blockIdx.x;
    const int64_t r0 = chunk * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
    for (int cg = lt; cg < C4; cg += tpr) {
        double s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0};
        float mean[4] = {0, 0, 0, 0}, inv[4] = {0, 0, 0, 0};
        if (MODE == 2) {
            float4 m = __ldg(reinterpret_cast<const float4*>(stats) + cg);
            float4 iv = __ldg(reinterpret_cast<const float4*>(stats + C) + cg);
            mean[0] = m.x; mean[1] = m.y; mean[2] = m.z; mean[3] = m.w;
            inv[0] = iv.x; inv[1] = iv.y; inv[2] = iv.z; inv[3] = iv.w;
        }
        auto accum = [&](const float4& q, const float4& gq) {
            float v[4] = {q.x, q.y, q.z, q.w};
            if (MODE == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) s0[j] += v[j];
            } else if (MODE == 1) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    s0[j] += v[j];
                    s1[j] += (double)v[j] * (double)v[j];
                }
            } else {
                float gv[4] = {gq.x, gq.y, gq.z, gq.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    double xhat = ((double)v[j] - (double)mean[j]) * (double)inv[j];
                    s0[j] += gv[j];
                    s1[j] += (double)gv[j] * xhat;
                }
            }
        };
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int64_t r = r0 + rr;
        // 4 rows in flight per thread (independent 128-bit loads), then the tail
        for (; r + 3 * rpi < r1; r += 4 * rpi) {
            float4 q[4], gq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                q[u] = __ldg(reinterpret_cast<const float4*>(x + (r + u * rpi) * C) + cg);
                gq[u] = MODE == 2 ? __ldg(reinterpret_cast<const float4*>(g + (r + u * rpi) * C) + cg) : zero4;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) accum(q[u], gq[u]);
        }
        for (; r < r1; r += rpi)
            accum(__ldg(reinterpret_cast<const float4*>(x + r * C) + cg),
                  MODE == 2 ? __ldg(reinterpret_cast<const float4*>(g + r * C) + cg) : zero4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            red[0][threadIdx.x][j] = s0[j];
            red[1][threadIdx.x][j] = s1[j];
        }
        __syncthreads();
        if (rr == 0) {
            for (int k = 1; k < rpi; ++k)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    s0[j] += red[0][k * tpr + lt][j];
                    s1[j] += red[1][k * tpr + lt][j];
                }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                part[(chunk * 2 + 0) * C + cg * 4 + j] = s0[j];
                part[(chunk * 2 + 1) * C + cg * 4 + j] = s1[j];
            }
        }
        __syncthreads();
    }
}

// Parallel fold of the per-chunk partials: block (32 columns x 16 chunk lanes),
// fixed order (lane-strided chunks, then a 16-way tree) -> deterministic.
template <int MODE>
__global__ void col_final2_k(const double* __restrict__ part, int64_t chunks, int64_t C, int64_t rows, double eps,
                             float* __restrict__ out0, float* __restrict__ out1) {
    __shared__ double sh[2][16][33];
    const int64_t col = blockIdx.x * 32 + threadIdx.x;
    double s0 = 0, s1 = 0;
    if (col < C)
        for (int64_t k = threadIdx.y; k < chunks; k += 16) {
            s0 += part[(k * 2 + 0) * C + col];
            s1 += part[(k * 2 + 1) * C + col];
        }
    sh[0][threadIdx.y][threadIdx.x] = s0;
    sh[1][threadIdx.y][threadIdx.x] = s1;
    __syncthreads();
    if (threadIdx.y != 0 || col >= C) return;
    for (int k = 1; k < 16; ++k) {
        s0 += sh[0][k][threadIdx.x];
        s1 += sh[1][k][threadIdx.x];
    }
    if (MODE == 0) {
        out0[col] = (float)s0;
    } else if (MODE == 1) {
        double mean = s0 / (double)rows;
        double var = s1 / (double)rows - mean * mean;
        if (var < 0) var = 0;
        out0[col] = (float)mean;
        out0[C + col] = (float)(1.0 / sqrt(var + eps));
    } else {
        out0[col] = (float)s0;
        out1[col] = (float)s1;
    }
}

template <int MODE>
__global__ void col_final_k(const double* __restrict__ part, int64_t chunks, int64_t C, int64_t rows, double eps,
                            float* __restrict__ out0, float* __restrict__ out1) {
    int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (col >= C) return;
    double s0 = 0, s1 = 0;
    for (int64_t k = 0; k < chunks; ++k) {
        s0 += part[(k * 2 + 0) * C + col];
        s1 += part[(k * 2 + 1) * C + col];
    }
    if (MODE == 0) {
        out0[col] = (float)s0;
    } else if (MODE == 1) {  // BN statistics: mean, 1/sqrt(var + eps), biased variance
        double mean = s0 / (double)rows;
        double var = s1 / (double)rows - mean * mean;
        if (var < 0) var = 0;
        out0[col] = (float)mean;
        out0[C + col] = (float)(1.0 / sqrt(var + eps));
    } else {
        out0[col] = (float)s0;
        out1[col] = (float)s1;
    }
}


template <int MODE>
int col_reduce(nncb_ctx* ctx, const float* x, const float* g, const float* stats, int64_t rows, int64_t C, double eps,
               float* out0, float* out1) {
    if (C <= 0) return 0;
    int64_t col_tiles = (C + 31) / 32;
    // enough chunks to fill ~4 waves of 148 SMs, at least 256 rows per chunk
    int64_t target = (int64_t)ctx->sm_count * 8;
    int64_t chunks = target / col_tiles;
    if (chunks < 1) chunks = 1;
    int64_t max_chunks = (rows + 255) / 256;
    if (chunks > max_chunks) chunks = max_chunks;
    if (chunks > 65535) chunks = 65535;
    if (chunks < 1) chunks = 1;
    int64_t rpc = (rows + chunks - 1) / chunks;
    // col_partial4_k (float4 rows) measured slower than the scalar 32x8 tiles on
    // every ResNet-50 shape; kept behind NNCB_COL_VEC=1 for experiments
    static const int vec = getenv("NNCB_COL_VEC") ? atoi(getenv("NNCB_COL_VEC")) : 0;
    if (vec == 1 && C % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        (!g || (reinterpret_cast<uintptr_t>(g) & 15) == 0) && (!stats || (reinterpret_cast<uintptr_t>(stats) & 15) == 0)) {
        int64_t ch4 = std::min<int64_t>((int64_t)ctx->sm_count * 8, std::max<int64_t>(1, rows / 64));
        int64_t rpc4 = (rows + ch4 - 1) / ch4;
        double* part = static_cast<double*>(nncb::scratch(ctx, sizeof(double) * 2 * ch4 * C));
        if (!part) return nncb::fail("col_reduce: scratch allocation failed");
        col_partial4_k<MODE><<<(unsigned)ch4, 256, 0, ctx->stream>>>(x, g, stats, part, rows, C, rpc4);
        NNCB_LAUNCHED(ctx);
        col_final2_k<MODE><<<(unsigned)((C + 31) / 32), dim3(32, 16), 0, ctx->stream>>>(part, ch4, C, rows, eps, out0,
                                                                                     out1);
        NNCB_LAUNCHED(ctx);
        return 0;
    }
    double* part = static_cast<double*>(nncb::scratch(ctx, sizeof(double) * 2 * chunks * C));
    if (!part) return nncb::fail("col_reduce: scratch allocation failed");
    dim3 grid((unsigned)col_tiles, (unsigned)chunks);
    col_partial_k<MODE><<<grid, dim3(32, 8), 0, ctx->stream>>>(x, g, stats, part, rows, C, rpc);
    NNCB_LAUNCHED(ctx);
    col_final2_k<MODE><<<(unsigned)((C + 31) / 32), dim3(32, 16), 0, ctx->stream>>>(part, chunks, C, rows, eps, out0,
                                                                                 out1);
    NNCB_LAUNCHED(ctx);
    return 0;
}

__global__ void sum_rows_exact_k(const float* __restrict__ x, float* __restrict__ out, int64_t rows, int64_t C) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C) return;
    float acc = 0.f;
    for (int64_t r = 0; r < rows; ++r) acc = __fadd_rn(acc, __ldg(x + r * C + c));
    out[c] = acc;
}

__global__ void bn_finalize_k(const double* __restrict__ cs, float* __restrict__ stats, int64_t rows, int64_t C,
                              double eps) {
    nncb::pdl_wait();   // launched as a programmatic dependent of the producing GEMM / reduction
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C) return;
    // (the same expression, uncontracted, as the GEMM's folded finalize: gemm_tc.cu bn_stats_from_sums)
    const double mean = __ddiv_rn(cs[c], (double)rows);
    double var = __dsub_rn(__ddiv_rn(cs[C + c], (double)rows), __dmul_rn(mean, mean));
    if (var < 0) var = 0;
    stats[c] = (float)mean;
    stats[C + c] = (float)__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, eps)));
}

// colstats from a materialized output (used when the GEMM ran on the exact
// path): cs[c] = sum_r y, cs[C+c] = sum_r y^2, in double. Chunk y of the rows
// writes its partials to part[y][2C] (block (32, 8), rows strided by 8 within
// the chunk, the 8 row sums folded in order); colstats_fold_k adds the chunks
// in order -- deterministic, no atomics.
__global__ void colstats_k(const float* __restrict__ y, double* __restrict__ part, int64_t rows, int64_t C,
                           int64_t rpc) {
    const int64_t c = blockIdx.x * 32 + threadIdx.x;
    const int64_t r0 = blockIdx.y * rpc, r1 = min(rows, r0 + rpc);
    double s0 = 0, s1 = 0;
    if (c < C)
        for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
            const double v = y[r * C + c];
            s0 += v;
            s1 += v * v;
        }
    __shared__ double sh[2][8][33];
    sh[0][threadIdx.y][threadIdx.x] = s0;
    sh[1][threadIdx.y][threadIdx.x] = s1;
    __syncthreads();
    if (threadIdx.y != 0 || c >= C) return;
    for (int k = 1; k < 8; ++k) {
        s0 += sh[0][k][threadIdx.x];
        s1 += sh[1][k][threadIdx.x];
    }
    part[blockIdx.y * 2 * C + c] = s0;
    part[blockIdx.y * 2 * C + C + c] = s1;
}

__global__ void colstats_fold_k(const double* __restrict__ part, int64_t chunks, int64_t C, double* __restrict__ cs) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C) return;
    double s0 = 0, s1 = 0;
    for (int64_t k = 0; k < chunks; ++k) {
        s0 += part[k * 2 * C + c];
        s1 += part[k * 2 * C + C + c];
    }
    cs[c] = s0;
    cs[C + c] = s1;
}

__global__ void cumsum_k(const float* __restrict__ x, float* __restrict__ y, int64_t outer, int64_t len, int64_t inner,
                         int exclusive, int reverse) {
    int64_t lines = outer * inner;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < lines; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = t / inner, in = t % inner;
        const float* xs = x + o * len * inner + in;
        float* ys = y + o * len * inner + in;
        float acc = 0.f;
        for (int64_t k = 0; k < len; ++k) {
            int64_t i = reverse ? len - 1 - k : k;
            if (exclusive) {
                ys[i * inner] = acc;
                acc = __fadd_rn(acc, xs[i * inner]);
            } else {
                acc = __fadd_rn(acc, xs[i * inner]);
                ys[i * inner] = acc;
            }
        }
    }
}

// LayerNorm: one CTA (256 threads) per row; row statistics in double.
template <int MODE>  // 0: forward, 1: backward dx, 2: row stats only
__global__ void __launch_bounds__(256) layernorm_k(const float* __restrict__ x, const float* __restrict__ gamma,
                                                   const float* __restrict__ beta, const float* __restrict__ gy,
                                                   float* __restrict__ out, float* __restrict__ row_stats, int64_t C,
                                                   double eps) {
    int64_t row = blockIdx.x;
    const float* xr = x + row * C;
    __shared__ double red[2][8];
    double s0 = 0, s1 = 0;
    for (int64_t c = threadIdx.x; c < C; c += 256) {
        double v = xr[c];
        s0 += v;
        s1 += v * v;
    }
    for (int o = 16; o; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (lane == 0) {
        red[0][warp] = s0;
        red[1][warp] = s1;
    }
    __syncthreads();
    s0 = 0;
    s1 = 0;
    for (int k = 0; k < 8; ++k) {
        s0 += red[0][k];
        s1 += red[1][k];
    }
    double mean_d = s0 / (double)C;
    double var = s1 / (double)C - mean_d * mean_d;
    if (var < 0) var = 0;
    float mean = (float)mean_d;
    float rstd = (float)(1.0 / sqrt(var + eps));
    if (MODE == 2) {
        if (threadIdx.x == 0) {
            row_stats[row * 2] = mean;
            row_stats[row * 2 + 1] = rstd;
        }
        return;
    }
    if (MODE == 0) {
        for (int64_t c = threadIdx.x; c < C; c += 256) {
            float xhat = __fmul_rn(__fsub_rn(xr[c], mean), rstd);
            out[row * C + c] = __fadd_rn(__fmul_rn(xhat, gamma[c]), beta[c]);
        }
        return;
    }
    // backward: gg = g*gamma; s1' = sum gg, s2' = sum gg*xhat
    const float* gr = gy + row * C;
    __syncthreads();
    double t0 = 0, t1 = 0;
    for (int64_t c = threadIdx.x; c < C; c += 256) {
        float xhat = __fmul_rn(__fsub_rn(xr[c], mean), rstd);
        float gg = __fmul_rn(gr[c], gamma[c]);
        t0 += gg;
        t1 += (double)gg * (double)xhat;
    }
    for (int o = 16; o; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
    }
    if (lane == 0) {
        red[0][warp] = t0;
        red[1][warp] = t1;
    }
    __syncthreads();
    t0 = 0;
    t1 = 0;
    for (int k = 0; k < 8; ++k) {
        t0 += red[0][k];
        t1 += red[1][k];
    }
    float sg = (float)t0, sgx = (float)t1, cnt = (float)C;
    for (int64_t c = threadIdx.x; c < C; c += 256) {
        float xhat = __fmul_rn(__fsub_rn(xr[c], mean), rstd);
        float gg = __fmul_rn(gr[c], gamma[c]);
        float t = __fadd_rn(sg, __fmul_rn(xhat, sgx));
        float u = __fsub_rn(gg, __fdiv_rn(t, cnt));
        out[row * C + c] = __fmul_rn(rstd, u);
    }
}

// LayerNorm with the row held in registers: VPT float4 per thread (C = 1024*VPT
// or less, C % 4 == 0), one global read of x (and g), float partial sums per
// thread folded in double. Same per-element arithmetic as layernorm_k.
template <int MODE, int VPT>
__global__ void __launch_bounds__(256) layernorm_reg_k(const float* __restrict__ x, const float* __restrict__ gamma,
                                                       const float* __restrict__ beta, const float* __restrict__ gy,
                                                       float* __restrict__ out, float* __restrict__ row_stats, int C,
                                                       double eps) {
    const int64_t row = blockIdx.x;
    const float4* xr = reinterpret_cast<const float4*>(x + row * C);
    const int C4 = C >> 2;
    __shared__ double red[2][8];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    auto block_sum2 = [&](double a, double b, double& ra, double& rb) {
        for (int o = 16; o; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        __syncthreads();
        if (lane == 0) {
            red[0][warp] = a;
            red[1][warp] = b;
        }
        __syncthreads();
        ra = 0;
        rb = 0;
        for (int k = 0; k < 8; ++k) {
            ra += red[0][k];
            rb += red[1][k];
        }
    };
    float4 v[VPT];
    float f0 = 0.f, f1 = 0.f;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int c4 = threadIdx.x + 256 * k;
        v[k] = c4 < C4 ? __ldg(xr + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        f0 += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        f1 += (v[k].x * v[k].x + v[k].y * v[k].y) + (v[k].z * v[k].z + v[k].w * v[k].w);
    }
    double s0, s1;
    block_sum2(f0, f1, s0, s1);
    const double mean_d = s0 / (double)C;
    double var = s1 / (double)C - mean_d * mean_d;
    if (var < 0) var = 0;
    const float mean = (float)mean_d;
    const float rstd = (float)(1.0 / sqrt(var + eps));
    if (MODE == 2) {
        if (threadIdx.x == 0) {
            row_stats[row * 2] = mean;
            row_stats[row * 2 + 1] = rstd;
        }
        return;
    }
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    float4* o4 = reinterpret_cast<float4*>(out + row * C);
    if (MODE == 0) {
        const float4* b4 = reinterpret_cast<const float4*>(beta);
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const int c4 = threadIdx.x + 256 * k;
            if (c4 >= C4) continue;
            const float4 ga = __ldg(g4 + c4), be = __ldg(b4 + c4);
            float4 y;
            y.x = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v[k].x, mean), rstd), ga.x), be.x);
            y.y = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v[k].y, mean), rstd), ga.y), be.y);
            y.z = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v[k].z, mean), rstd), ga.z), be.z);
            y.w = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v[k].w, mean), rstd), ga.w), be.w);
            o4[c4] = y;
        }
        return;
    }
    // backward: gg = g*gamma; sums of gg and gg*xhat, then dx
    const float4* gr = reinterpret_cast<const float4*>(gy + row * C);
    float4 gg[VPT];
    float t0f = 0.f, t1f = 0.f;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int c4 = threadIdx.x + 256 * k;
        if (c4 >= C4) {
            gg[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
        const float4 gv = __ldg(gr + c4), ga = __ldg(g4 + c4);
        gg[k] = make_float4(__fmul_rn(gv.x, ga.x), __fmul_rn(gv.y, ga.y), __fmul_rn(gv.z, ga.z), __fmul_rn(gv.w, ga.w));
        const float xh[4] = {__fmul_rn(__fsub_rn(v[k].x, mean), rstd), __fmul_rn(__fsub_rn(v[k].y, mean), rstd),
                             __fmul_rn(__fsub_rn(v[k].z, mean), rstd), __fmul_rn(__fsub_rn(v[k].w, mean), rstd)};
        t0f += (gg[k].x + gg[k].y) + (gg[k].z + gg[k].w);
        t1f += (gg[k].x * xh[0] + gg[k].y * xh[1]) + (gg[k].z * xh[2] + gg[k].w * xh[3]);
    }
    double t0, t1;
    block_sum2(t0f, t1f, t0, t1);
    const float sg = (float)t0, sgx = (float)t1, cnt = (float)C, inv_cnt = 1.f / cnt;
    const bool pow2 = (C & (C - 1)) == 0;   // t / C as an exact-reciprocal product (same rounding)
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int c4 = threadIdx.x + 256 * k;
        if (c4 >= C4) continue;
        const float vv[4] = {v[k].x, v[k].y, v[k].z, v[k].w}, gq[4] = {gg[k].x, gg[k].y, gg[k].z, gg[k].w};
        float r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float xhat = __fmul_rn(__fsub_rn(vv[j], mean), rstd);
            const float t = __fadd_rn(sg, __fmul_rn(xhat, sgx));
            r[j] = __fmul_rn(rstd, __fsub_rn(gq[j], pow2 ? __fmul_rn(t, inv_cnt) : __fdiv_rn(t, cnt)));
        }
        o4[c4] = make_float4(r[0], r[1], r[2], r[3]);
    }
}

template <int MODE>
bool layernorm_reg(nncb_ctx* ctx, const float* x, const float* gamma, const float* beta, const float* g, float* out,
                   float* rs, int64_t rows, int64_t C, double eps) {
    static const bool off = getenv("NNCB_LN_REG") && atoi(getenv("NNCB_LN_REG")) == 0;
    if (off || C % 4 != 0 || C > 8192) return false;
    for (const void* p : {(const void*)x, (const void*)gamma, (const void*)beta, (const void*)g, (const void*)out})
        if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return false;
    const int vpt = static_cast<int>((C / 4 + 255) / 256);
    const unsigned grid = static_cast<unsigned>(rows);
    const int Ci = static_cast<int>(C);
    if (vpt <= 1)
        layernorm_reg_k<MODE, 1><<<grid, 256, 0, ctx->stream>>>(x, gamma, beta, g, out, rs, Ci, eps);
    else if (vpt <= 2)
        layernorm_reg_k<MODE, 2><<<grid, 256, 0, ctx->stream>>>(x, gamma, beta, g, out, rs, Ci, eps);
    else if (vpt <= 4)
        layernorm_reg_k<MODE, 4><<<grid, 256, 0, ctx->stream>>>(x, gamma, beta, g, out, rs, Ci, eps);
    else
        layernorm_reg_k<MODE, 8><<<grid, 256, 0, ctx->stream>>>(x, gamma, beta, g, out, rs, Ci, eps);
    return true;
}

// LayerNorm backward with the parameter gradients folded in (tensor-core
// modes): besides dx (identical per row to layernorm_reg_k<1>), every CTA
// accumulates, for the rows it owns, the per-column sums
//   dgamma_c = sum_r g[r,c] * xhat[r,c]    dbeta_c = sum_r g[r,c]
// in double registers (each thread owns the same VPT*4 columns in every row)
// and writes them once as partials[cta][2][C]; ln_param_final_k folds the
// partials in CTA order, so the result is deterministic. Replaces the row
// statistics pass + column pass of nncb_layernorm_dgamma and the SumRows of
// the beta gradient (reference semantics: src/nnc/graph/op.cpp LayerNorm
// extension; CPU restatement oracle/restated64.py node_vjp LayerNorm).
// LayerNorm backward with the parameter gradients folded in (tensor-core
// modes): besides dx (bitwise identical per row to layernorm_reg_k<1>), every
// CTA accumulates, over the rows it owns (row = blockIdx.x + k*gridDim.x, at
// most kLnRowsPerCta of them), the per-column sums
//   dgamma_c = sum_r g[r,c] * xhat[r,c]    dbeta_c = sum_r g[r,c]
// in a float shared-memory array (each thread owns the same columns in every
// row, so the read-modify-write needs no atomics) and stores them once as
// partials[cta][2][C]; ln_param_final_k folds the partials in double in CTA
// order, so the result is deterministic. Replaces the row statistics pass and
// the column pass of nncb_layernorm_dgamma and the SumRows of the beta
// gradient (CPU restatement: oracle/restated64.py node_vjp LayerNorm).
constexpr int64_t kLnRowsPerCta = 256;

template <int VPT>
__global__ void __launch_bounds__(256, VPT > 4 ? 2 : 4)
    layernorm_bwd_acc_k(const float* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ gy,
                        float* __restrict__ out, float* __restrict__ part, int64_t rows, int C, double eps) {
    extern __shared__ __align__(16) float4 acc[];   // [dgamma | dbeta][C4]
    __shared__ double red[2][8];
    const int C4 = C >> 2;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    auto block_sum2 = [&](double a, double b, double& ra, double& rb) {
        for (int o = 16; o; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        __syncthreads();
        if (lane == 0) {
            red[0][warp] = a;
            red[1][warp] = b;
        }
        __syncthreads();
        ra = 0;
        rb = 0;
        for (int k = 0; k < 8; ++k) {
            ra += red[0][k];
            rb += red[1][k];
        }
    };
    for (int c4 = threadIdx.x; c4 < 2 * C4; c4 += 256) acc[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    // t / C: a multiplication by the exact reciprocal when C is a power of two
    // (the same correctly rounded result as the division)
    const bool pow2 = (C & (C - 1)) == 0;
    const float cnt = (float)C, inv_cnt = 1.f / cnt;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const float4* xr = reinterpret_cast<const float4*>(x + row * C);
        const float4* gr = reinterpret_cast<const float4*>(gy + row * C);
        float4 v[VPT], gv[VPT];
        float f0 = 0.f, f1 = 0.f;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const int c4 = threadIdx.x + 256 * k;
            const bool in = c4 < C4;
            v[k] = in ? __ldg(xr + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
            gv[k] = in ? __ldcs(gr + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
            f0 += (v[k].x + v[k].y) + (v[k].z + v[k].w);
            f1 += (v[k].x * v[k].x + v[k].y * v[k].y) + (v[k].z * v[k].z + v[k].w * v[k].w);
        }
        double s0, s1;
        block_sum2(f0, f1, s0, s1);
        const double mean_d = s0 / (double)C;
        double var = s1 / (double)C - mean_d * mean_d;
        if (var < 0) var = 0;
        const float mean = (float)mean_d;
        const float rstd = (float)(1.0 / sqrt(var + eps));
        float t0f = 0.f, t1f = 0.f;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const int c4 = threadIdx.x + 256 * k;
            if (c4 >= C4) continue;
            const float4 ga = __ldg(g4 + c4);
            const float gg[4] = {__fmul_rn(gv[k].x, ga.x), __fmul_rn(gv[k].y, ga.y), __fmul_rn(gv[k].z, ga.z),
                                 __fmul_rn(gv[k].w, ga.w)};
            const float xh[4] = {__fmul_rn(__fsub_rn(v[k].x, mean), rstd), __fmul_rn(__fsub_rn(v[k].y, mean), rstd),
                                 __fmul_rn(__fsub_rn(v[k].z, mean), rstd), __fmul_rn(__fsub_rn(v[k].w, mean), rstd)};
            t0f += (gg[0] + gg[1]) + (gg[2] + gg[3]);
            t1f += (gg[0] * xh[0] + gg[1] * xh[1]) + (gg[2] * xh[2] + gg[3] * xh[3]);
        }
        double t0, t1;
        block_sum2(t0f, t1f, t0, t1);
        const float sg = (float)t0, sgx = (float)t1;
        float4* o4 = reinterpret_cast<float4*>(out + row * C);
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const int c4 = threadIdx.x + 256 * k;
            if (c4 >= C4) continue;
            const float4 ga = __ldg(g4 + c4);
            const float vv[4] = {v[k].x, v[k].y, v[k].z, v[k].w}, graw[4] = {gv[k].x, gv[k].y, gv[k].z, gv[k].w},
                        gam[4] = {ga.x, ga.y, ga.z, ga.w};
            float r[4], ax[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float xhat = __fmul_rn(__fsub_rn(vv[j], mean), rstd);
                const float t = __fadd_rn(sg, __fmul_rn(xhat, sgx));
                r[j] = __fmul_rn(rstd, __fsub_rn(__fmul_rn(graw[j], gam[j]), pow2 ? __fmul_rn(t, inv_cnt) : __fdiv_rn(t, cnt)));
                ax[j] = graw[j] * xhat;
            }
            __stcs(o4 + c4, make_float4(r[0], r[1], r[2], r[3]));
            float4 a = acc[c4], b = acc[C4 + c4];
            a.x += ax[0]; a.y += ax[1]; a.z += ax[2]; a.w += ax[3];
            b.x += graw[0]; b.y += graw[1]; b.z += graw[2]; b.w += graw[3];
            acc[c4] = a;
            acc[C4 + c4] = b;
        }
    }
    float4* p4 = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * 2 * C);
    __syncthreads();   // the dbeta half of acc is owned by other threads when C4 % 256 != 0
    for (int c4 = threadIdx.x; c4 < 2 * C4; c4 += 256) p4[c4] = acc[c4];
}

// Fold of the per-CTA partials in two fixed-order levels (deterministic):
// ln_param_fold_k: block (32, 8), grid (column quads / 32, kLnFoldSplits);
// thread (tx, ty) of split s sums, in double, the chunks ty, ty+8, ... of
// split s for four columns; the eight row sums are added in ty order into
// part2[s][2][C]. ln_param_final_k adds the splits in order.
constexpr int kLnFoldSplits = 16;

__global__ void ln_param_fold_k(const float* __restrict__ part, int64_t chunks, int64_t C, double* __restrict__ part2) {
    const int64_t C4 = C >> 2, q = blockIdx.x * 32 + threadIdx.x;
    const int64_t per = (chunks + kLnFoldSplits - 1) / kLnFoldSplits;
    const int64_t k0 = blockIdx.y * per, k1 = min(chunks, k0 + per);
    __shared__ double sh[8][8][33];
    double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (q < C4) {
        const float4* p4 = reinterpret_cast<const float4*>(part);
#pragma unroll 2
        for (int64_t k = k0 + threadIdx.y; k < k1; k += 8) {
            const float4 u = __ldcs(p4 + (k * 2 + 0) * C4 + q), w = __ldcs(p4 + (k * 2 + 1) * C4 + q);
            a[0] += u.x; a[1] += u.y; a[2] += u.z; a[3] += u.w;
            a[4] += w.x; a[5] += w.y; a[6] += w.z; a[7] += w.w;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) sh[j][threadIdx.y][threadIdx.x] = a[j];
    __syncthreads();
    if (threadIdx.y != 0 || q >= C4) return;
    for (int k = 1; k < 8; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += sh[j][k][threadIdx.x];
    double* o = part2 + (int64_t)blockIdx.y * 2 * C;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        o[q * 4 + j] = a[j];
        o[C + q * 4 + j] = a[4 + j];
    }
}

__global__ void ln_param_final_k(const double* __restrict__ part2, int64_t C, float* __restrict__ dgamma,
                                 float* __restrict__ dbeta) {
    const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (col >= C) return;
    double s0 = 0, s1 = 0;
    for (int k = 0; k < kLnFoldSplits; ++k) {
        s0 += part2[(int64_t)k * 2 * C + col];
        s1 += part2[(int64_t)k * 2 * C + C + col];
    }
    if (dgamma) dgamma[col] = (float)s0;
    if (dbeta) dbeta[col] = (float)s1;
}

__global__ void ln_dgamma_partial_k(const float* __restrict__ x, const float* __restrict__ g,
                                    const float* __restrict__ rs, double* __restrict__ part, int64_t rows, int64_t C,
                                    int64_t rpc) {
    int64_t col = blockIdx.x * 32 + threadIdx.x;
    int64_t chunk = blockIdx.y;
    int64_t r0 = chunk * rpc, r1 = min(rows, r0 + rpc);
    double s = 0;
    if (col < C)
        for (int64_t r = r0 + threadIdx.y; r < r1; r += blockDim.y) {
            float xhat = __fmul_rn(__fsub_rn(x[r * C + col], rs[r * 2]), rs[r * 2 + 1]);
            s += (double)g[r * C + col] * (double)xhat;
        }
    __shared__ double sh[8][33];
    sh[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && col < C) {
        for (int k = 1; k < (int)blockDim.y; ++k) s += sh[k][threadIdx.x];
        part[(chunk * 2) * C + col] = s;
        part[(chunk * 2 + 1) * C + col] = 0;
    }
}

__global__ void l1_k(const float* __restrict__ p, const float* __restrict__ t, float* __restrict__ grad,
                     double* __restrict__ partial, int64_t n) {
    double inv = n > 0 ? 1.0 / (double)n : 0.0;
    double acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    auto one = [&](float pv, float tv) -> float {
        const double d = __dsub_rn((double)pv, (double)tv);
        acc = __dadd_rn(acc, fabs(d));
        return (float)(d > 0 ? inv : (d < 0 ? -inv : 0.0));
    };
    const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(t) |
                       reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    int64_t tail = 0;
    if (vec) {   // float4 body; the gradient element values are unchanged
        const int64_t n4 = n / 4;
        for (int64_t i = t0; i < n4; i += stride) {
            const float4 pv = __ldg(reinterpret_cast<const float4*>(p) + i);
            const float4 tv = __ldg(reinterpret_cast<const float4*>(t) + i);
            float4 gv;
            gv.x = one(pv.x, tv.x);
            gv.y = one(pv.y, tv.y);
            gv.z = one(pv.z, tv.z);
            gv.w = one(pv.w, tv.w);
            reinterpret_cast<float4*>(grad)[i] = gv;
        }
        tail = n4 * 4;
    }
    for (int64_t i = tail + t0; i < n; i += stride) grad[i] = one(p[i], t[i]);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double red[32];
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0;
        for (int k = 0; k < (int)(blockDim.x / 32); ++k) s += red[k];
        partial[blockIdx.x] = s;
    }
}

__global__ void l1_final_k(const double* __restrict__ partial, int blocks, int64_t n, double* __restrict__ loss) {
    if (threadIdx.x != 0) return;
    double s = 0;
    for (int k = 0; k < blocks; ++k) s += partial[k];
    *loss = s * (n > 0 ? 1.0 / (double)n : 0.0);
}

// Softmax cross-entropy over the last axis (extension loss; CPU restatement
// oracle/restated64.py softmax_ce): per row r of logits z[r, 0:C] with
// probability-vector targets t, loss_r = -sum_c t_c (z_c - m - log s),
// s = sum_c exp(z_c - m), m = max_c z_c, and grad = (exp(z - m)/s - t)/rows.
// One CTA per row; the row's max, exp-sum and loss are reduced in double in a
// fixed tree (deterministic), the rows' losses summed in order by one thread.
template <int THREADS>
__device__ __forceinline__ double block_reduce_d(double v, double* sh, bool is_max) {
    for (int o = 16; o; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, u) : v + u;
    }
    __syncthreads();
    if (threadIdx.x % 32 == 0) sh[threadIdx.x / 32] = v;
    __syncthreads();
    double r = sh[0];
    for (int k = 1; k < THREADS / 32; ++k) r = is_max ? fmax(r, sh[k]) : r + sh[k];
    return r;
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) softmax_ce_row_k(const float* __restrict__ z, const float* __restrict__ t,
                                                             float* __restrict__ grad, double* __restrict__ row_loss,
                                                             int64_t C, double inv_rows) {
    __shared__ double sh[THREADS / 32];
    const int64_t r = blockIdx.x;
    const float* zr = z + r * C;
    const float* tr = t + r * C;
    double m = -INFINITY;
    for (int64_t c = threadIdx.x; c < C; c += THREADS) m = fmax(m, (double)zr[c]);
    m = block_reduce_d<THREADS>(m, sh, true);
    double se = 0, tz = 0, ts = 0;
    for (int64_t c = threadIdx.x; c < C; c += THREADS) {
        const double d = (double)zr[c] - m;
        se += exp(d);
        tz += (double)tr[c] * d;
        ts += (double)tr[c];
    }
    se = block_reduce_d<THREADS>(se, sh, false);
    tz = block_reduce_d<THREADS>(tz, sh, false);
    ts = block_reduce_d<THREADS>(ts, sh, false);
    const double ls = log(se);
    for (int64_t c = threadIdx.x; c < C; c += THREADS)
        grad[r * C + c] = (float)((exp((double)zr[c] - m) / se - (double)tr[c]) * inv_rows);
    if (threadIdx.x == 0) row_loss[r] = ts * ls - tz;   // -sum t (d - log s)
}

__global__ void softmax_ce_final_k(const double* __restrict__ row_loss, int64_t rows, double* __restrict__ loss) {
    if (threadIdx.x != 0) return;
    double s = 0;
    for (int64_t r = 0; r < rows; ++r) s += row_loss[r];
    *loss = rows > 0 ? s / (double)rows : 0.0;
}

// (float)((double)w - lr*(double)g) with separately rounded double ops, exactly
// runtime.cpp:493 (no FMA contraction).
__device__ __forceinline__ float sgd1(float w, float g, double lr, double scale) {
    return (float)__dsub_rn((double)w, __dmul_rn(lr, __dmul_rn((double)g, scale)));
}

// lr read from device memory (a captured step graph stays valid across learning-rate changes)
__global__ void sgd_dev_k(float* __restrict__ w, const float* __restrict__ g, int64_t n,
                          const double* __restrict__ lr_dev, double scale) {
    const double lr = *lr_dev;
    int64_t nv = n >> 2;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        float4 wv = reinterpret_cast<float4*>(w)[v];
        float4 gv = __ldg(reinterpret_cast<const float4*>(g) + v);
        wv.x = sgd1(wv.x, gv.x, lr, scale);
        wv.y = sgd1(wv.y, gv.y, lr, scale);
        wv.z = sgd1(wv.z, gv.z, lr, scale);
        wv.w = sgd1(wv.w, gv.w, lr, scale);
        reinterpret_cast<float4*>(w)[v] = wv;
    }
    for (int64_t i = (nv << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        w[i] = sgd1(w[i], g[i], lr, scale);
}

__global__ void sgd_k(float* __restrict__ w, const float* __restrict__ g, int64_t n, double lr, double scale) {
    int64_t nv = n >> 2;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        float4 wv = reinterpret_cast<float4*>(w)[v];
        float4 gv = __ldg(reinterpret_cast<const float4*>(g) + v);
        wv.x = sgd1(wv.x, gv.x, lr, scale);
        wv.y = sgd1(wv.y, gv.y, lr, scale);
        wv.z = sgd1(wv.z, gv.z, lr, scale);
        wv.w = sgd1(wv.w, gv.w, lr, scale);
        reinterpret_cast<float4*>(w)[v] = wv;
    }
    for (int64_t i = (nv << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        w[i] = sgd1(w[i], g[i], lr, scale);
}

}  // namespace

namespace nncb {
int colstats_from_output(nncb_ctx* ctx, const float* y, double* cs, int64_t rows, int64_t C) {
    if (C <= 0) return 0;
    const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(1024, (rows + 255) / 256));
    const int64_t rpc = (rows + chunks - 1) / chunks;
    double* part = static_cast<double*>(scratch(ctx, sizeof(double) * 2 * C * chunks));
    if (!part) return fail("colstats: scratch allocation failed");
    colstats_k<<<dim3((unsigned)((C + 31) / 32), (unsigned)chunks), dim3(32, 8), 0, ctx->stream>>>(y, part, rows, C, rpc);
    NNCB_LAUNCHED(ctx);
    colstats_fold_k<<<(unsigned)((C + 127) / 128), 128, 0, ctx->stream>>>(part, chunks, C, cs);
    NNCB_LAUNCHED(ctx);
    return 0;
}
}  // namespace nncb

extern "C" {

int nncb_maxpool_fwd(nncb_ctx* ctx, const nncb_pool_geom* g, const float* x, float* y, float* idx) {
    int64_t total = g->n * g->oh * g->ow * g->c;
    if (total == 0) return 0;
    const bool k33 = g->kh == 3 && g->kw == 3 && g->sh == 2 && g->sw == 2 && g->c % 4 == 0 &&
                     std::max(total, g->n * g->ih * g->iw * g->c) < (int64_t(1) << 31);
    if (k33)
        maxpool_fwd_k33<<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(x, y, idx, *g);
    else if (g->c % 4 == 0)
        maxpool_fwd_k<4><<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(x, y, idx, *g);
    else
        maxpool_fwd_k<1><<<nncb::grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(x, y, idx, *g);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_maxpool_bwd(nncb_ctx* ctx, const nncb_pool_geom* g, const float* idx, const float* gy, float* gx) {
    int64_t total = g->n * g->ih * g->iw * g->c;
    if (total == 0) return 0;
    const int64_t out_total = g->n * g->oh * g->ow * g->c;
    const bool i32 = std::max(total, out_total) < (int64_t(1) << 31);   // 32-bit index decode when it fits
    if (g->c % 4 == 0 && i32)
        if (g->kh == 3 && g->kw == 3 && g->sh == 2 && g->sw == 2)
            maxpool_bwd_k33<<<nncb::grid_for(ctx, total / 16, 256), 256, 0, ctx->stream>>>(idx, gy, gx, *g);
        else
            maxpool_bwd_k<4, int><<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(idx, gy, gx, *g);
    else if (g->c % 4 == 0)
        maxpool_bwd_k<4, int64_t><<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(idx, gy, gx, *g);
    else if (i32)
        maxpool_bwd_k<1, int><<<nncb::grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(idx, gy, gx, *g);
    else
        maxpool_bwd_k<1, int64_t><<<nncb::grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(idx, gy, gx, *g);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_avgpool_fwd(nncb_ctx* ctx, int64_t n, int64_t ih, int64_t iw, int64_t c, int64_t oh, int64_t ow,
                     const float* x, float* y) {
    int64_t total = n * oh * ow * c;
    if (total == 0) return 0;
    if (oh == 1 && ow == 1 && c % 4 == 0 && n * ih * iw * c < (int64_t(1) << 31) &&
        !((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)) {
        const float scale = 1.0f / static_cast<float>(ih * iw);   // = __fdiv_rn(1, window) of the general kernel
        avgpool_fwd_global4_k<<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(
            x, y, static_cast<uint32_t>(ih * iw), static_cast<uint32_t>(c / 4), static_cast<uint32_t>(total / 4), scale);
        NNCB_LAUNCHED(ctx);
        return 0;
    }
    avgpool_fwd_k<<<nncb::grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(x, y, n, ih, iw, c, oh, ow);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_avgpool_bwd(nncb_ctx* ctx, int64_t n, int64_t ih, int64_t iw, int64_t c, int64_t oh, int64_t ow,
                     const float* gy, float* gx) {
    int64_t total = n * ih * iw * c;
    if (total == 0) return 0;
    const bool i32 = std::max(total, n * oh * ow * c) < (int64_t(1) << 31);
    if (oh == 1 && ow == 1 && c % 4 == 0 && i32)
        avgpool_bwd_global_k<<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(
            gy, gx, static_cast<uint32_t>(ih * iw), static_cast<uint32_t>(c / 4), static_cast<uint32_t>(total / 4));
    else if (c % 4 == 0 && i32)
        avgpool_bwd_k<4, int><<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(gy, gx, n, ih, iw, c, oh, ow);
    else if (c % 4 == 0)
        avgpool_bwd_k<4, int64_t><<<nncb::grid_for(ctx, total / 4, 256), 256, 0, ctx->stream>>>(gy, gx, n, ih, iw, c, oh, ow);
    else if (i32)
        avgpool_bwd_k<1, int><<<nncb::grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(gy, gx, n, ih, iw, c, oh, ow);
    else
        avgpool_bwd_k<1, int64_t><<<nncb::grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(gy, gx, n, ih, iw, c, oh, ow);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_sum_rows(nncb_ctx* ctx, const float* x, float* out, int64_t rows, int64_t cols, int exact) {
    if (!exact) return col_reduce<0>(ctx, x, nullptr, nullptr, rows, cols, 0.0, out, nullptr);
    if (cols == 0) return 0;
    sum_rows_exact_k<<<(unsigned)((cols + 127) / 128), 128, 0, ctx->stream>>>(x, out, rows, cols);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_cumsum(nncb_ctx* ctx, const float* x, float* y, int64_t outer, int64_t len, int64_t inner, int exclusive,
                int reverse) {
    int64_t lines = outer * inner;
    if (lines == 0 || len == 0) return 0;
    cumsum_k<<<nncb::grid_for(ctx, lines, 128), 128, 0, ctx->stream>>>(x, y, outer, len, inner, exclusive, reverse);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_bn_stats(nncb_ctx* ctx, const float* x, float* stats, int64_t rows, int64_t C, double eps) {
    return col_reduce<1>(ctx, x, nullptr, nullptr, rows, C, eps, stats, nullptr);
}

namespace {
__global__ void colsums_to_float_k(const double* __restrict__ s, float* __restrict__ o0, float* __restrict__ o1,
                                   int64_t C) {
    nncb::pdl_wait();
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < C) {
        o0[c] = static_cast<float>(s[c]);
        o1[c] = static_cast<float>(s[C + c]);
    }
}
}  // namespace

int nncb_colsums_to_float(nncb_ctx* ctx, const double* sums, float* out0, float* out1, int64_t C) {
    if (C <= 0) return 0;
    NNCB_CUDA(nncb::launch_pdl(colsums_to_float_k, dim3((unsigned)((C + 255) / 256)), dim3(256), ctx->stream, sums, out0,
                               out1, C));
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_bn_finalize(nncb_ctx* ctx, const double* colstats, float* stats, int64_t rows, int64_t C, double eps) {
    if (C <= 0) return 0;
    NNCB_CUDA(nncb::launch_pdl(bn_finalize_k, dim3((unsigned)((C + 127) / 128)), dim3(128), ctx->stream, colstats, stats,
                               rows, C, eps));
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_bn_grad_reduce(nncb_ctx* ctx, const float* x, const float* stats, const float* g, float* sum_g,
                        float* sum_gx, int64_t rows, int64_t C) {
    return col_reduce<2>(ctx, x, g, stats, rows, C, 0.0, sum_g, sum_gx);
}

int nncb_layernorm_fwd(nncb_ctx* ctx, const float* x, const float* gamma, const float* beta, float* y, int64_t rows,
                       int64_t C, double eps) {
    if (rows == 0) return 0;
    if (!layernorm_reg<0>(ctx, x, gamma, beta, nullptr, y, nullptr, rows, C, eps))
        layernorm_k<0><<<(unsigned)rows, 256, 0, ctx->stream>>>(x, gamma, beta, nullptr, y, nullptr, C, eps);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_layernorm_bwd(nncb_ctx* ctx, const float* x, const float* gamma, const float* g, float* gx, int64_t rows,
                       int64_t C, double eps) {
    if (rows == 0) return 0;
    if (!layernorm_reg<1>(ctx, x, gamma, nullptr, g, gx, nullptr, rows, C, eps))
        layernorm_k<1><<<(unsigned)rows, 256, 0, ctx->stream>>>(x, gamma, nullptr, g, gx, nullptr, C, eps);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_layernorm_bwd_params(nncb_ctx* ctx, const float* x, const float* gamma, const float* g, float* gx,
                              float* dgamma, float* dbeta, int64_t rows, int64_t C, double eps) {
    if (!dgamma && !dbeta) return nncb_layernorm_bwd(ctx, x, gamma, g, gx, rows, C, eps);
    if (rows == 0) {
        if (dgamma) cudaMemsetAsync(dgamma, 0, sizeof(float) * C, ctx->stream);
        if (dbeta) cudaMemsetAsync(dbeta, 0, sizeof(float) * C, ctx->stream);
        return 0;
    }
    bool aligned = C % 4 == 0 && C <= 8192;
    for (const void* p : {(const void*)x, (const void*)gamma, (const void*)g, (const void*)gx})
        aligned = aligned && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
    if (!aligned) {   // unfused sequence
        if (int rc = nncb_layernorm_bwd(ctx, x, gamma, g, gx, rows, C, eps)) return rc;
        if (dgamma)
            if (int rc = nncb_layernorm_dgamma(ctx, x, g, dgamma, rows, C, eps)) return rc;
        if (dbeta)
            if (int rc = nncb_sum_rows(ctx, g, dbeta, rows, C, 0)) return rc;
        return 0;
    }
    const int vpt = static_cast<int>((C / 4 + 255) / 256);
    const int Ci = static_cast<int>(C);
    const size_t smem = sizeof(float) * 2 * C;   // the CTA's dgamma / dbeta accumulators
    float* part = nullptr;
    double* part2 = nullptr;
    auto go = [&](auto kern) {
        // a full wave of resident CTAs, more when a CTA would own more than
        // kLnRowsPerCta rows (bounds the float accumulation length)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
        int64_t grid = std::max<int64_t>((int64_t)ctx->sm_count * std::max(per_sm, 1),
                                         (rows + kLnRowsPerCta - 1) / kLnRowsPerCta);
        if (grid > rows) grid = rows;
        const size_t p2 = (sizeof(float) * 2 * grid * C + 255) / 256 * 256;
        char* base = static_cast<char*>(nncb::scratch(ctx, p2 + sizeof(double) * 2 * kLnFoldSplits * C));
        if (!base) return (int64_t)0;
        part = reinterpret_cast<float*>(base);
        part2 = reinterpret_cast<double*>(base + p2);
        kern<<<static_cast<unsigned>(grid), 256, smem, ctx->stream>>>(x, gamma, g, gx, part, rows, Ci, eps);
        return grid;
    };
    int64_t grid;
    if (vpt <= 1)
        grid = go(layernorm_bwd_acc_k<1>);
    else if (vpt <= 2)
        grid = go(layernorm_bwd_acc_k<2>);
    else if (vpt <= 4)
        grid = go(layernorm_bwd_acc_k<4>);
    else
        grid = go(layernorm_bwd_acc_k<8>);
    if (!grid) return nncb::fail("layernorm_bwd_params: scratch allocation failed");
    NNCB_LAUNCHED(ctx);
    ln_param_fold_k<<<dim3((unsigned)((C / 4 + 31) / 32), kLnFoldSplits), dim3(32, 8), 0, ctx->stream>>>(part, grid, C,
                                                                                                       part2);
    NNCB_LAUNCHED(ctx);
    ln_param_final_k<<<(unsigned)((C + 127) / 128), 128, 0, ctx->stream>>>(part2, C, dgamma, dbeta);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_layernorm_dgamma(nncb_ctx* ctx, const float* x, const float* g, float* dgamma, int64_t rows, int64_t C,
                          double eps) {
    if (rows == 0) return 0;
    int64_t col_tiles = (C + 31) / 32;
    int64_t chunks = ((int64_t)ctx->sm_count * 8) / col_tiles;
    if (chunks < 1) chunks = 1;
    if (chunks > (rows + 63) / 64) chunks = (rows + 63) / 64;
    if (chunks < 1) chunks = 1;
    int64_t rpc = (rows + chunks - 1) / chunks;
    size_t stats_bytes = sizeof(float) * 2 * rows;
    size_t part_off = (stats_bytes + 255) / 256 * 256;
    char* base = static_cast<char*>(nncb::scratch(ctx, part_off + sizeof(double) * 2 * chunks * C));
    if (!base) return nncb::fail("layernorm_dgamma: scratch allocation failed");
    float* rs = reinterpret_cast<float*>(base);
    double* part = reinterpret_cast<double*>(base + part_off);
    if (!layernorm_reg<2>(ctx, x, nullptr, nullptr, nullptr, nullptr, rs, rows, C, eps))
        layernorm_k<2><<<(unsigned)rows, 256, 0, ctx->stream>>>(x, nullptr, nullptr, nullptr, nullptr, rs, C, eps);
    NNCB_LAUNCHED(ctx);
    ln_dgamma_partial_k<<<dim3((unsigned)col_tiles, (unsigned)chunks), dim3(32, 8), 0, ctx->stream>>>(x, g, rs, part,
                                                                                                      rows, C, rpc);
    NNCB_LAUNCHED(ctx);
    col_final_k<0><<<(unsigned)((C + 127) / 128), 128, 0, ctx->stream>>>(part, chunks, C, rows, 0.0, dgamma, nullptr);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_l1_loss(nncb_ctx* ctx, const float* pred, const float* target, float* grad, double* loss_dev, int64_t n) {
    const int threads = 256;
    unsigned blocks = nncb::grid_for(ctx, n, threads, 2);
    double* partial = static_cast<double*>(nncb::scratch(ctx, sizeof(double) * blocks));
    if (!partial) return nncb::fail("l1_loss: scratch allocation failed");
    l1_k<<<blocks, threads, 0, ctx->stream>>>(pred, target, grad, partial, n);
    NNCB_LAUNCHED(ctx);
    l1_final_k<<<1, 32, 0, ctx->stream>>>(partial, (int)blocks, n, loss_dev);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_softmax_ce(nncb_ctx* ctx, const float* logits, const float* target, float* grad, double* loss_dev,
                    int64_t rows, int64_t C) {
    if (rows <= 0 || C <= 0) return nncb::fail("nncb_softmax_ce: empty logits");
    if (rows > (int64_t(1) << 31) - 1) return nncb::fail("nncb_softmax_ce: too many rows");
    double* row_loss = static_cast<double*>(nncb::scratch(ctx, sizeof(double) * static_cast<size_t>(rows)));
    if (!row_loss) return nncb::fail("softmax_ce: scratch allocation failed");
    softmax_ce_row_k<256><<<(unsigned)rows, 256, 0, ctx->stream>>>(logits, target, grad, row_loss, C, 1.0 / (double)rows);
    NNCB_LAUNCHED(ctx);
    softmax_ce_final_k<<<1, 32, 0, ctx->stream>>>(row_loss, rows, loss_dev);
    NNCB_LAUNCHED(ctx);
    return 0;
}

// SGD over several element ranges of the flat regions in one launch:
// blockIdx.y picks the range (ranges[2r] offset, ranges[2r+1] count, both in
// elements, offsets 16-byte aligned), blockIdx.x strides within it.
__global__ void sgd_ranges_k(float* __restrict__ w, const float* __restrict__ g, const int64_t* __restrict__ ranges,
                             const double* __restrict__ lr_dev, double scale) {
    const double lr = *lr_dev;
    const int64_t off = ranges[2 * blockIdx.y], n = ranges[2 * blockIdx.y + 1];
    float* wr = w + off;
    const float* gr = g + off;
    const int64_t nv = n >> 2, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += stride) {
        float4 wv = reinterpret_cast<float4*>(wr)[v];
        const float4 gv = __ldg(reinterpret_cast<const float4*>(gr) + v);
        wv.x = sgd1(wv.x, gv.x, lr, scale);
        wv.y = sgd1(wv.y, gv.y, lr, scale);
        wv.z = sgd1(wv.z, gv.z, lr, scale);
        wv.w = sgd1(wv.w, gv.w, lr, scale);
        reinterpret_cast<float4*>(wr)[v] = wv;
    }
    for (int64_t i = (nv << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        wr[i] = sgd1(wr[i], gr[i], lr, scale);
}

int nncb_sgd(nncb_ctx* ctx, float* w, const float* g, int64_t n, double lr, double grad_scale) {
    if (n <= 0) return 0;
    if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g)) & 15)
        return nncb::fail("nncb_sgd: buffers must be 16-byte aligned");
    sgd_k<<<nncb::grid_for(ctx, (n + 3) / 4, 256), 256, 0, ctx->stream>>>(w, g, n, lr, grad_scale);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_sgd_dev_ranges(nncb_ctx* ctx, int stream, float* w, const float* g, const int64_t* ranges_dev,
                        int n_ranges, int64_t max_count, const double* lr_dev, double grad_scale) {
    if (n_ranges <= 0) return 0;
    if (n_ranges > 65535) return nncb::fail("nncb_sgd_dev_ranges: too many ranges");
    const unsigned gx = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(64, (max_count / 4 + 255) / 256)));
    sgd_ranges_k<<<dim3(gx, static_cast<unsigned>(n_ranges)), 256, 0, nncb::stream_of(ctx, stream)>>>(
        w, g, ranges_dev, lr_dev, grad_scale);
    NNCB_LAUNCHED(ctx);
    return 0;
}

int nncb_sgd_dev(nncb_ctx* ctx, int stream, float* w, const float* g, int64_t n, const double* lr_dev,
                 double grad_scale) {
    if (n <= 0) return 0;
    if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g)) & 15)
        return nncb::fail("nncb_sgd_dev: buffers must be 16-byte aligned");
    sgd_dev_k<<<nncb::grid_for(ctx, (n + 3) / 4, 256), 256, 0, nncb::stream_of(ctx, stream)>>>(w, g, n, lr_dev,
                                                                                              grad_scale);
    NNCB_LAUNCHED(ctx);
    return 0;
}

}  // extern "C"
