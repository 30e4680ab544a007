"""The bf16 tensor-core path (NNCB_PREC_BF16: tcgen05.mma kind::f16 on bf16
operand copies, fp32 accumulation in TMEM) at the kernel level: forward and
input-gradient contractions of dense layers and convolutions, and dense
weight gradients (over transposed bf16 copies), against float64
products of the same bf16-rounded operands (what remains is fp32 accumulation
order), asserting through nncb_gemm_last_path that the tensor-core path ran;
shapes the route does not take (convolution weight gradients, narrow K blocks,
memory-bound contractions below the intensity threshold) run tf32, and are
checked against tf32-truncated operands."""
import ctypes

import numpy as np
import pytest

from oracle import restated64 as R64
from tests.nncb_ctypes import Dev, GemmDesc, K, ctx

pytestmark = pytest.mark.gpu
BF16 = 2


def bf16(a):
    """Round to nearest even at bf16 (8-bit mantissa), back to float64."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def run(desc, A, B, out_shape, bias=None):
    Ad, Bd = Dev(A), Dev(B)
    Od = Dev(nbytes=int(np.prod(out_shape)) * 4)
    bd = Dev(bias) if bias is not None else None
    rc = K.nncb_gemm(ctx(), ctypes.byref(desc), Ad.p, Bd.p, bd.p if bd else None, Od.p)
    assert rc == 0, K.nncb_last_error()
    assert K.nncb_gemm_last_path() == 1
    K.nncb_sync(ctx())
    return Od.get(out_shape).astype(np.float64)


def operand(a, route):
    """The operand as the device multiplies it: bf16-rounded on the bf16 route,
    tf32-truncated on the tf32 one (R64.bf16_route mirrors the device rule)."""
    return bf16(a) if R64.bf16_route(*route) else R64.tf32_trunc(a)


def rel(got, want):
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30))


@pytest.mark.parametrize("batch,fin,fout", [(512, 1024, 256), (8192, 4096, 4096), (100, 72, 40), (256, 2048, 1024)])
def test_dense_fwd_and_dgrad_bf16(batch, fin, fout):
    rng = np.random.default_rng(batch + fin)
    x = rng.uniform(-1, 1, (batch, fin)).astype(np.float32)
    w = rng.uniform(-1, 1, (fin, fout)).astype(np.float32)
    b = rng.uniform(-1, 1, fout).astype(np.float32)
    y = run(GemmDesc(kind=0, precision=BF16, epilogue=1, batch=batch, in_f=fin, out_f=fout), x, w, (batch, fout), b)
    rf = (fin, fin, fout, "fwd", 1)
    assert rel(y, operand(x, rf) @ operand(w, rf) + b) < 1e-5
    assert rel(y, x.astype(np.float64) @ w + b) < 2e-2          # against the exact product
    g = rng.uniform(-1, 1, (batch, fout)).astype(np.float32)
    gx = run(GemmDesc(kind=1, precision=BF16, batch=batch, in_f=fin, out_f=fout), g, w, (batch, fin))
    rd = (fout, fout, fin, "dgrad", 1)
    assert rel(gx, operand(g, rd) @ operand(w, rd).T) < 1e-5


@pytest.mark.parametrize("n,h,ci,co,k,s", [(8, 14, 256, 256, 3, 1), (4, 28, 128, 512, 1, 1), (4, 56, 64, 64, 3, 1),
                                            (2, 28, 128, 128, 3, 2)])
def test_conv_fwd_and_dgrad_bf16(n, h, ci, co, k, s):
    rng = np.random.default_rng(n * h + ci)
    x = rng.uniform(-1, 1, (n, h, h, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32) / np.sqrt(k * k * ci)
    oh, ow, ph, pw = R64.conv_geom(x.shape, (k, k), (s, s), True)
    geo = dict(n=n, ih=h, iw=h, ci=ci, co=co, kh=k, kw=k, sh=s, sw=s, oh=oh, ow=ow, pad_top=ph[0], pad_left=pw[0])
    y = run(GemmDesc(kind=3, precision=BF16, **geo), x, w, (n, oh, ow, co))
    rf = (k * k * ci, ci, co, "fwd", k * k)
    assert rel(y, R64.conv2d(operand(x, rf), operand(w, rf), None, (s, s), True)) < 1e-5
    g = rng.uniform(-1, 1, (n, oh, ow, co)).astype(np.float32)
    gx = run(GemmDesc(kind=4, precision=BF16, **geo), g, w, (n, h, h, ci))
    rd = (k * k * co, co, ci, "dgrad", k * k)
    assert rel(gx, R64.conv2d_grad_input(operand(g, rd), operand(w, rd), x.shape, (s, s), True)) < 1e-5


@pytest.mark.parametrize("batch,fin,fout", [(8192, 4096, 4096), (256, 2048, 1000)])
def test_dense_wgrad_bf16_over_transposed_copies(batch, fin, fout):
    """dW = x^T g as the forward contraction of K-major bf16 transposes."""
    rng = np.random.default_rng(fin)
    x = rng.uniform(-1, 1, (batch, fin)).astype(np.float32)
    g = rng.uniform(-1, 1, (batch, fout)).astype(np.float32)
    gw = run(GemmDesc(kind=2, precision=BF16, batch=batch, in_f=fin, out_f=fout), x, g, (fin, fout))
    rw = (batch, fin, fout, "dense_wgrad", 1)
    assert rel(gw, operand(x, rw).T @ operand(g, rw)) < 3e-5   # (a 8192-long fp32 accumulation)


def test_wgrad_runs_tf32_under_bf16_precision():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (4, 14, 14, 64)).astype(np.float32)
    g = rng.uniform(-1, 1, (4, 14, 14, 64)).astype(np.float32)
    geo = dict(n=4, ih=14, iw=14, ci=64, co=64, kh=3, kw=3, sh=1, sw=1, oh=14, ow=14, pad_top=1, pad_left=1)
    gw = run(GemmDesc(kind=5, precision=BF16, **geo), x, g, (3, 3, 64, 64))
    want = R64.conv2d_grad_weight(R64.tf32_trunc(x), R64.tf32_trunc(g), (3, 3, 64, 64), (1, 1), True)
    assert rel(gw, want) < 1e-5
