"""The tcgen05 tf32 implicit-GEMM convolutions (forward, input gradient,
weight gradient) directly against the float64 CPU restatement
(oracle/restated64.py conv2d / conv2d_grad_input / conv2d_grad_weight, itself
pinned to the reference run in float64) fed the operands truncated to tf32
exactly as kind::tf32 reads them, at batch 32-64 and ResNet-50 channel counts
(ci % 32 == 0: the TMA / halo / sub-pixel-phase / split-K routes). What is
left is fp32 accumulation order: 1e-5 of max|y|. Reference kernels:
kernels.hpp:166-243."""
import numpy as np
import pytest

from oracle import restated64 as R64
from tests.nncb_ctypes import Dev, GemmDesc, K, gemm
from tests.test_gpu_gemm import CONV_DGRAD, CONV_FWD, CONV_WGRAD, conv_geom

pytestmark = pytest.mark.gpu

SHAPES = [  # n, h(=w), ci, co, k, s
    (64, 14, 256, 256, 3, 1),   # stage-2 3x3 (halo patches)
    (32, 28, 128, 512, 1, 1),   # stage-1 expansion 1x1
    (32, 56, 64, 64, 3, 1),     # stage-0 3x3, N = 64
    (64, 28, 128, 128, 3, 2),   # strided 3x3 (sub-pixel dgrad phases)
    (64, 7, 512, 2048, 1, 1),   # stage-3 expansion
    (32, 56, 256, 512, 1, 2),   # strided projection
]


def rel(got, want):
    return float(np.max(np.abs(got.astype(np.float64) - want)) / max(np.max(np.abs(want)), 1e-30))


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind", ["fwd", "dgrad", "wgrad"])
def test_tf32_conv_against_float64_oracle(shape, kind):
    n, h, ci, co, k, s = shape
    g = conv_geom(n, h, h, ci, co, k, s)
    rng = np.random.default_rng(n + h + ci + co + k + s)
    x = rng.uniform(-1, 1, (n, h, h, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    xt, wt, gt = R64.tf32_trunc(x), R64.tf32_trunc(w), R64.tf32_trunc(gy)
    if kind == "fwd":
        d = GemmDesc(kind=CONV_FWD, precision=0, **g)
        out = Dev(nbytes=gy.nbytes)
        gemm(d, Dev(x), Dev(w), None, out)
        got, want = out.get(gy.shape), R64.conv2d(xt, wt, None, (s, s), True)
    elif kind == "dgrad":
        d = GemmDesc(kind=CONV_DGRAD, precision=0, **g)
        out = Dev(nbytes=x.nbytes)
        gemm(d, Dev(gy), Dev(w), None, out)
        got, want = out.get(x.shape), R64.conv2d_grad_input(gt, wt, x.shape, (s, s), True)
    else:
        d = GemmDesc(kind=CONV_WGRAD, precision=0, **g)
        out = Dev(nbytes=w.nbytes)
        gemm(d, Dev(x), Dev(gy), None, out)
        got, want = out.get(w.shape), R64.conv2d_grad_weight(xt, gt, w.shape, (s, s), True)
    assert K.nncb_gemm_last_path() == 1, "tensor-core path not taken"
    e = rel(got, want)
    assert e < 1e-5, e
