/* oracle/nnc_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference CPU kernels on the hot path, plus the extension ops the reference
 * does not have. Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
 * may load it (as oracle/_ref/libnnc_oracle.so), never the product.
 *
 * Reference-vocabulary kernels restate /root/reference/proj/core/include/nnc/
 * kernels.hpp loop by loop (same summation order, separately rounded products;
 * built with -ffp-contract=off) and are pinned bit-exact against the reference
 * itself in tests/test_oracle.py:
 *   relu / relu_grad / add / mul      kernels.hpp:47-70
 *   dense, dense_grad_input/_weight   kernels.hpp:118-151, sum_cols :153-160
 *   conv2d, conv2d_grad_input/_weight kernels.hpp:166-243, sum_nhw :245-250
 *   maxpool2d(+grad)                  kernels.hpp:258-302
 *   adaptive_avg_pool2d(+grad)        kernels.hpp:304-344
 *   l1_loss, sgd                      runtime.cpp:468-496
 * Extension ops (PARITY UNPINNED by the reference -- it has none of them):
 *   batchnorm (training statistics / inference moving statistics), gelu (erf),
 *   layernorm, and their gradients. Formulas are the textbook ones; the float
 *   operation order of each "apply" step is the one the B200 kernels use, and
 *   statistics are accumulated in double.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef int64_t i64;

/* geometry: TF-SAME / VALID (kernels.cpp:12-53) */
typedef struct { i64 n, ih, iw, ci, co, kh, kw, sh, sw, oh, ow, pt, pl; } geom_t;

void o_relu(const float* x, float* y, i64 n) { for (i64 i = 0; i < n; ++i) y[i] = x[i] > 0.f ? x[i] : 0.f; }
void o_relu_grad(const float* x, const float* g, float* y, i64 n) {
    for (i64 i = 0; i < n; ++i) y[i] = x[i] > 0.f ? g[i] : 0.f;
}
void o_add(const float* a, const float* b, float* y, i64 n) { for (i64 i = 0; i < n; ++i) y[i] = a[i] + b[i]; }
void o_mul(const float* a, const float* b, float* y, i64 n) { for (i64 i = 0; i < n; ++i) y[i] = a[i] * b[i]; }

void o_dense(const float* x, const float* w, const float* bias, float* y, i64 batch, i64 in, i64 out) {
    for (i64 b = 0; b < batch; ++b)
        for (i64 o = 0; o < out; ++o) {
            float acc = bias ? bias[o] : 0.f;
            for (i64 i = 0; i < in; ++i) acc += x[b * in + i] * w[i * out + o];
            y[b * out + o] = acc;
        }
}

void o_dense_grad_input(const float* g, const float* w, float* gx, i64 batch, i64 in, i64 out) {
    for (i64 b = 0; b < batch; ++b)
        for (i64 i = 0; i < in; ++i) {
            float acc = 0.f;
            for (i64 o = 0; o < out; ++o) acc += g[b * out + o] * w[i * out + o];
            gx[b * in + i] = acc;
        }
}

void o_dense_grad_weight(const float* x, const float* g, float* gw, i64 batch, i64 in, i64 out) {
    for (i64 i = 0; i < in; ++i)
        for (i64 o = 0; o < out; ++o) {
            float acc = 0.f;
            for (i64 b = 0; b < batch; ++b) acc += x[b * in + i] * g[b * out + o];
            gw[i * out + o] = acc;
        }
}

void o_sum_cols(const float* g, float* gb, i64 batch, i64 out) {
    for (i64 o = 0; o < out; ++o) {
        float acc = 0.f;
        for (i64 b = 0; b < batch; ++b) acc += g[b * out + o];
        gb[o] = acc;
    }
}

void o_conv2d(const float* x, const float* k, const float* bias, float* y, const geom_t* g) {
    for (i64 n = 0; n < g->n; ++n)
        for (i64 oh = 0; oh < g->oh; ++oh)
            for (i64 ow = 0; ow < g->ow; ++ow)
                for (i64 co = 0; co < g->co; ++co) {
                    float acc = bias ? bias[co] : 0.f;
                    for (i64 dh = 0; dh < g->kh; ++dh) {
                        i64 h = oh * g->sh + dh - g->pt;
                        if (h < 0 || h >= g->ih) continue;
                        for (i64 dw = 0; dw < g->kw; ++dw) {
                            i64 w = ow * g->sw + dw - g->pl;
                            if (w < 0 || w >= g->iw) continue;
                            const float* xp = x + ((n * g->ih + h) * g->iw + w) * g->ci;
                            const float* kp = k + ((dh * g->kw + dw) * g->ci) * g->co + co;
                            for (i64 ci = 0; ci < g->ci; ++ci) acc += xp[ci] * kp[ci * g->co];
                        }
                    }
                    y[((n * g->oh + oh) * g->ow + ow) * g->co + co] = acc;
                }
}

void o_conv2d_grad_input(const float* gy, const float* k, float* gx, const geom_t* g) {
    memset(gx, 0, sizeof(float) * g->n * g->ih * g->iw * g->ci);
    for (i64 n = 0; n < g->n; ++n)
        for (i64 oh = 0; oh < g->oh; ++oh)
            for (i64 ow = 0; ow < g->ow; ++ow) {
                const float* gp = gy + ((n * g->oh + oh) * g->ow + ow) * g->co;
                for (i64 dh = 0; dh < g->kh; ++dh) {
                    i64 h = oh * g->sh + dh - g->pt;
                    if (h < 0 || h >= g->ih) continue;
                    for (i64 dw = 0; dw < g->kw; ++dw) {
                        i64 w = ow * g->sw + dw - g->pl;
                        if (w < 0 || w >= g->iw) continue;
                        float* xp = gx + ((n * g->ih + h) * g->iw + w) * g->ci;
                        const float* kp = k + ((dh * g->kw + dw) * g->ci) * g->co;
                        for (i64 ci = 0; ci < g->ci; ++ci) {
                            float acc = 0.f;
                            for (i64 co = 0; co < g->co; ++co) acc += gp[co] * kp[ci * g->co + co];
                            xp[ci] += acc;
                        }
                    }
                }
            }
}

void o_conv2d_grad_weight(const float* x, const float* gy, float* gk, const geom_t* g) {
    memset(gk, 0, sizeof(float) * g->kh * g->kw * g->ci * g->co);
    for (i64 n = 0; n < g->n; ++n)
        for (i64 oh = 0; oh < g->oh; ++oh)
            for (i64 ow = 0; ow < g->ow; ++ow) {
                const float* gp = gy + ((n * g->oh + oh) * g->ow + ow) * g->co;
                for (i64 dh = 0; dh < g->kh; ++dh) {
                    i64 h = oh * g->sh + dh - g->pt;
                    if (h < 0 || h >= g->ih) continue;
                    for (i64 dw = 0; dw < g->kw; ++dw) {
                        i64 w = ow * g->sw + dw - g->pl;
                        if (w < 0 || w >= g->iw) continue;
                        const float* xp = x + ((n * g->ih + h) * g->iw + w) * g->ci;
                        float* kp = gk + ((dh * g->kw + dw) * g->ci) * g->co;
                        for (i64 ci = 0; ci < g->ci; ++ci)
                            for (i64 co = 0; co < g->co; ++co) kp[ci * g->co + co] += xp[ci] * gp[co];
                    }
                }
            }
}

void o_sum_nhw(const float* gy, float* gb, i64 rows, i64 c) {
    memset(gb, 0, sizeof(float) * c);
    for (i64 i = 0; i < rows; ++i)
        for (i64 ch = 0; ch < c; ++ch) gb[ch] += gy[i * c + ch];
}

/* pool geometry: n, ih, iw, c, kh, kw, sh, sw, oh, ow */
void o_maxpool2d(const float* x, float* y, float* idx, const i64* p) {
    i64 N = p[0], IH = p[1], IW = p[2], C = p[3], KH = p[4], KW = p[5], SH = p[6], SW = p[7], OH = p[8], OW = p[9];
    for (i64 n = 0; n < N; ++n)
        for (i64 oh = 0; oh < OH; ++oh)
            for (i64 ow = 0; ow < OW; ++ow)
                for (i64 c = 0; c < C; ++c) {
                    float best = 0.f;
                    i64 bi = -1;
                    for (i64 dh = 0; dh < KH; ++dh)
                        for (i64 dw = 0; dw < KW; ++dw) {
                            float v = x[((n * IH + oh * SH + dh) * IW + ow * SW + dw) * C + c];
                            if (bi < 0 || v > best) {
                                best = v;
                                bi = dh * KW + dw;
                            }
                        }
                    i64 at = ((n * OH + oh) * OW + ow) * C + c;
                    y[at] = best;
                    if (idx) idx[at] = (float)bi;
                }
}

void o_maxpool2d_grad(const float* idx, const float* gy, float* gx, const i64* p) {
    i64 N = p[0], IH = p[1], IW = p[2], C = p[3], KW = p[5], SH = p[6], SW = p[7], OH = p[8], OW = p[9];
    memset(gx, 0, sizeof(float) * N * IH * IW * C);
    for (i64 n = 0; n < N; ++n)
        for (i64 oh = 0; oh < OH; ++oh)
            for (i64 ow = 0; ow < OW; ++ow)
                for (i64 c = 0; c < C; ++c) {
                    i64 at = ((n * OH + oh) * OW + ow) * C + c;
                    i64 wi = (i64)idx[at];
                    gx[((n * IH + oh * SH + wi / KW) * IW + ow * SW + wi % KW) * C + c] += gy[at];
                }
}

static i64 a_start(i64 o, i64 in, i64 out) { return (o * in) / out; }
static i64 a_end(i64 o, i64 in, i64 out) { return ((o + 1) * in + out - 1) / out; }

void o_avgpool(const float* x, float* y, i64 n, i64 ih, i64 iw, i64 c, i64 oh, i64 ow) {
    for (i64 b = 0; b < n; ++b)
        for (i64 o = 0; o < oh; ++o)
            for (i64 p = 0; p < ow; ++p) {
                i64 h0 = a_start(o, ih, oh), h1 = a_end(o, ih, oh), w0 = a_start(p, iw, ow), w1 = a_end(p, iw, ow);
                float scale = 1.f / (float)((h1 - h0) * (w1 - w0));
                for (i64 ch = 0; ch < c; ++ch) {
                    float acc = 0.f;
                    for (i64 h = h0; h < h1; ++h)
                        for (i64 w = w0; w < w1; ++w) acc += x[((b * ih + h) * iw + w) * c + ch];
                    y[((b * oh + o) * ow + p) * c + ch] = acc * scale;
                }
            }
}

void o_avgpool_grad(const float* gy, float* gx, i64 n, i64 ih, i64 iw, i64 c, i64 oh, i64 ow) {
    memset(gx, 0, sizeof(float) * n * ih * iw * c);
    for (i64 b = 0; b < n; ++b)
        for (i64 o = 0; o < oh; ++o)
            for (i64 p = 0; p < ow; ++p) {
                i64 h0 = a_start(o, ih, oh), h1 = a_end(o, ih, oh), w0 = a_start(p, iw, ow), w1 = a_end(p, iw, ow);
                float scale = 1.f / (float)((h1 - h0) * (w1 - w0));
                for (i64 ch = 0; ch < c; ++ch) {
                    float gv = gy[((b * oh + o) * ow + p) * c + ch] * scale;
                    for (i64 h = h0; h < h1; ++h)
                        for (i64 w = w0; w < w1; ++w) gx[((b * ih + h) * iw + w) * c + ch] += gv;
                }
            }
}

double o_l1_loss(const float* p, const float* t, float* grad, i64 n) {
    double inv = n > 0 ? 1.0 / (double)n : 0.0, acc = 0;
    for (i64 i = 0; i < n; ++i) {
        double d = (double)p[i] - (double)t[i];
        acc += fabs(d);
        grad[i] = (float)(d > 0 ? inv : (d < 0 ? -inv : 0.0));
    }
    return acc * inv;
}

void o_sgd(float* w, const float* g, i64 n, double lr) {
    for (i64 i = 0; i < n; ++i) w[i] = (float)((double)w[i] - lr * (double)g[i]);
}

/* ---------------- extension ops (parity unpinned) ---------------------- */

/* stats[0:C] = mean, stats[C:2C] = 1/sqrt(biased var + eps); double accumulation */
void o_bn_stats(const float* x, float* stats, i64 rows, i64 C, double eps) {
    for (i64 c = 0; c < C; ++c) {
        double s = 0, s2 = 0;
        for (i64 r = 0; r < rows; ++r) {
            double v = x[r * C + c];
            s += v;
            s2 += v * v;
        }
        double mean = s / (double)rows, var = s2 / (double)rows - mean * mean;
        if (var < 0) var = 0;
        stats[c] = (float)mean;
        stats[C + c] = (float)(1.0 / sqrt(var + eps));
    }
}

/* y = ((x - mean) * invstd) * gamma + beta, each step rounded to float */
void o_bn_apply(const float* x, const float* stats, const float* gamma, const float* beta, float* y, i64 rows, i64 C) {
    for (i64 r = 0; r < rows; ++r)
        for (i64 c = 0; c < C; ++c) {
            float t = (x[r * C + c] - stats[c]) * stats[C + c];
            y[r * C + c] = t * gamma[c] + beta[c];
        }
}

void o_bn_infer(const float* x, const float* mm, const float* mv, const float* gamma, const float* beta, float* y,
                i64 rows, i64 C, double eps) {
    for (i64 r = 0; r < rows; ++r)
        for (i64 c = 0; c < C; ++c) {
            float s = (float)(1.0 / sqrt((double)mv[c] + eps));
            float t = (x[r * C + c] - mm[c]) * s;
            y[r * C + c] = t * gamma[c] + beta[c];
        }
}

/* sum_g[c] = sum g, sum_gx[c] = sum g * xhat (double) */
void o_bn_grad_reduce(const float* x, const float* stats, const float* g, float* sum_g, float* sum_gx, i64 rows,
                      i64 C) {
    for (i64 c = 0; c < C; ++c) {
        double s0 = 0, s1 = 0;
        for (i64 r = 0; r < rows; ++r) {
            double xhat = ((double)x[r * C + c] - (double)stats[c]) * (double)stats[C + c];
            s0 += g[r * C + c];
            s1 += (double)g[r * C + c] * xhat;
        }
        sum_g[c] = (float)s0;
        sum_gx[c] = (float)s1;
    }
}

/* dx = (gamma*invstd) * (g - (sum_g + xhat*sum_gx)/M) */
void o_bn_grad_input(const float* x, const float* stats, const float* g, const float* gamma, const float* sum_g,
                     const float* sum_gx, float* dx, i64 rows, i64 C) {
    float cnt = (float)rows;
    for (i64 r = 0; r < rows; ++r)
        for (i64 c = 0; c < C; ++c) {
            float xhat = (x[r * C + c] - stats[c]) * stats[C + c];
            float t = sum_g[c] + xhat * sum_gx[c];
            float u = g[r * C + c] - t / cnt;
            dx[r * C + c] = (gamma[c] * stats[C + c]) * u;
        }
}

void o_gelu(const float* x, float* y, i64 n) {
    for (i64 i = 0; i < n; ++i) {
        double v = x[i];
        y[i] = (float)(0.5 * v * (1.0 + erf(v * 0.70710678118654752440)));
    }
}

void o_gelu_grad(const float* x, const float* g, float* y, i64 n) {
    for (i64 i = 0; i < n; ++i) {
        double v = x[i];
        double cdf = 0.5 * (1.0 + erf(v * 0.70710678118654752440));
        double pdf = exp(-0.5 * v * v) * 0.39894228040143267794;
        y[i] = (float)((double)g[i] * (cdf + v * pdf));
    }
}

static void ln_row_stats(const float* xr, i64 C, double eps, float* mean, float* rstd) {
    double s = 0, s2 = 0;
    for (i64 c = 0; c < C; ++c) {
        s += xr[c];
        s2 += (double)xr[c] * xr[c];
    }
    double m = s / (double)C, var = s2 / (double)C - m * m;
    if (var < 0) var = 0;
    *mean = (float)m;
    *rstd = (float)(1.0 / sqrt(var + eps));
}

void o_layernorm(const float* x, const float* gamma, const float* beta, float* y, i64 rows, i64 C, double eps) {
    for (i64 r = 0; r < rows; ++r) {
        float mean, rstd;
        ln_row_stats(x + r * C, C, eps, &mean, &rstd);
        for (i64 c = 0; c < C; ++c) {
            float xhat = (x[r * C + c] - mean) * rstd;
            y[r * C + c] = xhat * gamma[c] + beta[c];
        }
    }
}

void o_layernorm_grad_input(const float* x, const float* gamma, const float* g, float* dx, i64 rows, i64 C,
                            double eps) {
    for (i64 r = 0; r < rows; ++r) {
        float mean, rstd;
        ln_row_stats(x + r * C, C, eps, &mean, &rstd);
        double t0 = 0, t1 = 0;
        for (i64 c = 0; c < C; ++c) {
            float xhat = (x[r * C + c] - mean) * rstd;
            float gg = g[r * C + c] * gamma[c];
            t0 += gg;
            t1 += (double)gg * (double)xhat;
        }
        float sg = (float)t0, sgx = (float)t1, cnt = (float)C;
        for (i64 c = 0; c < C; ++c) {
            float xhat = (x[r * C + c] - mean) * rstd;
            float gg = g[r * C + c] * gamma[c];
            float t = sg + xhat * sgx;
            float u = gg - t / cnt;
            dx[r * C + c] = rstd * u;
        }
    }
}

void o_layernorm_dgamma(const float* x, const float* g, float* dgamma, i64 rows, i64 C, double eps) {
    for (i64 c = 0; c < C; ++c) dgamma[c] = 0;
    double* acc = (double*)__builtin_alloca(sizeof(double) * (C > 0 ? C : 1));
    for (i64 c = 0; c < C; ++c) acc[c] = 0;
    for (i64 r = 0; r < rows; ++r) {
        float mean, rstd;
        ln_row_stats(x + r * C, C, eps, &mean, &rstd);
        for (i64 c = 0; c < C; ++c) {
            float xhat = (x[r * C + c] - mean) * rstd;
            acc[c] += (double)g[r * C + c] * (double)xhat;
        }
    }
    for (i64 c = 0; c < C; ++c) dgamma[c] = (float)acc[c];
}
