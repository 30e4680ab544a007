"""Kernel-level GEMM tests: the tcgen05 tf32 path against the exact fp32 path
(bit-identical to the reference CPU loops) for all six contraction kinds,
strided / padded convolutions and ragged tile edges. Bound: 2e-2 of max|ref|
(reduced-precision GEMM tolerance); typical tf32 error is ~1e-3."""
import ctypes
import numpy as np
import pytest

from tests.nncb_ctypes import K, Dev, GemmDesc, ctx, gemm

pytestmark = pytest.mark.gpu

DENSE_FWD, DENSE_DGRAD, DENSE_WGRAD, CONV_FWD, CONV_DGRAD, CONV_WGRAD = range(6)


def conv_geom(n, ih, iw, ci, co, k, s, same=True):
    oh = -(-ih // s) if same else (ih - k) // s + 1
    ow = -(-iw // s) if same else (iw - k) // s + 1
    pt = max((oh - 1) * s + k - ih, 0) // 2 if same else 0
    pl = max((ow - 1) * s + k - iw, 0) // 2 if same else 0
    return dict(n=n, ih=ih, iw=iw, ci=ci, co=co, kh=k, kw=k, sh=s, sw=s, oh=oh, ow=ow, pad_top=pt, pad_left=pl)


def run_both(kind, geo, a, b, bias, out_shape, expect_tc=None):
    """tf32 tensor-core result and exact result; expect_tc=True asserts the
    tf32 request really ran on the tcgen05 kernel (no silent exact fallback)."""
    outs = []
    for prec in (0, 1):
        d = GemmDesc(kind=kind, precision=prec, epilogue=1 if bias is not None else 0, **geo)
        o = Dev(nbytes=int(np.prod(out_shape)) * 4)
        gemm(d, a, b, bias, o)   # a, b, bias are held by the caller
        if prec == 0 and expect_tc is not None:
            assert K.nncb_gemm_last_path() == int(expect_tc), "tensor-core path not taken"
        outs.append(o.get(out_shape))
    return outs


def check(tc, ex):
    err = np.max(np.abs(tc.astype(np.float64) - ex)) / max(np.max(np.abs(ex)), 1e-30)
    assert err < 2e-2, err
    return err


CONVS = [
    (2, 32, 32, 3, 64, 7, 2), (2, 16, 16, 16, 32, 3, 1),
    (2, 14, 14, 64, 64, 3, 1), (2, 13, 11, 64, 96, 3, 2), (4, 7, 7, 128, 256, 1, 1),
    (2, 16, 16, 32, 64, 1, 2), (1, 9, 9, 64, 32, 3, 2), (3, 8, 8, 96, 128, 3, 1),
    # channel counts below a 32-wide block: builder-warp (manual A) path
    (3, 19, 23, 3, 32, 3, 1), (2, 15, 15, 12, 64, 5, 2), (1, 30, 30, 4, 128, 7, 2),
    # stride-2 few-channel convs: space-to-depth route (odd sizes, SAME padding)
    (2, 17, 23, 3, 32, 7, 2), (1, 9, 9, 8, 16, 3, 2),
]


@pytest.mark.parametrize("shape", CONVS)
def test_conv_fwd(shape):
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    bias = rng.uniform(-1, 1, co).astype(np.float32)
    tc, ex = run_both(CONV_FWD, g, Dev(x), Dev(w), Dev(bias), (n, g["oh"], g["ow"], co), expect_tc=True)
    check(tc, ex)


@pytest.mark.parametrize("shape", CONVS)
def test_conv_dgrad(shape):
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(1)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    tc_ok = k == 1 or (ci % 32 == 0 and co % 32 == 0)
    tc, ex = run_both(CONV_DGRAD, g, Dev(gy), Dev(w), None, (n, ih, iw, ci), expect_tc=True if tc_ok else None)
    check(tc, ex)


@pytest.mark.parametrize("shape", CONVS)
def test_conv_wgrad(shape):
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    tc, ex = run_both(CONV_WGRAD, g, Dev(x), Dev(gy), None, (k, k, ci, co), expect_tc=True)
    check(tc, ex)


@pytest.mark.parametrize("b,i,o", [(32, 2048, 64), (256, 2048, 1000), (200, 96, 160), (64, 128, 16), (300, 148, 64)])
def test_dense(b, i, o):
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (b, i)).astype(np.float32)
    w = rng.uniform(-1, 1, (i, o)).astype(np.float32)
    bias = rng.uniform(-1, 1, o).astype(np.float32)
    gy = rng.uniform(-1, 1, (b, o)).astype(np.float32)
    geo = dict(batch=b, in_f=i, out_f=o)
    tc, ex = run_both(DENSE_FWD, geo, Dev(x), Dev(w), Dev(bias), (b, o))
    check(tc, ex)
    ref = x.astype(np.float64) @ w + bias
    assert np.max(np.abs(ex - ref)) / np.max(np.abs(ref)) < 1e-5
    tc, ex = run_both(DENSE_DGRAD, geo, Dev(gy), Dev(w), None, (b, i))
    check(tc, ex)
    tc, ex = run_both(DENSE_WGRAD, geo, Dev(x), Dev(gy), None, (i, o))
    check(tc, ex)


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("shape", [(2, 14, 14, 64, 64, 3, 1), (2, 32, 32, 3, 64, 7, 2), (3, 7, 7, 128, 96, 1, 1),
                                   (16, 28, 28, 128, 256, 1, 1)])
def test_conv_fwd_fused_column_statistics(shape, precision):
    """NNCB_EPI_COLSTATS: per-channel sum / sum of squares of the conv output
    accumulated in the tcgen05 epilogue (fixed-point integer atomics) or, on
    the exact path, by a deterministic pass over the output -- vs the output,
    and bitwise identical when the call is repeated."""
    import ctypes
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    xd, wd = Dev(x), Dev(w)
    cs = Dev(nbytes=2 * co * 8)
    out = Dev(nbytes=n * g["oh"] * g["ow"] * co * 4)
    d = GemmDesc(kind=CONV_FWD, precision=precision, epilogue=4, colstats=cs.p.value, **g)
    gemm(d, xd, wd, None, out)
    y = out.get((n * g["oh"] * g["ow"], co)).astype(np.float64)
    got = np.frombuffer(cs.get((4 * co,)).tobytes(), np.float64)
    assert np.allclose(got[:co], y.sum(0), rtol=1e-5, atol=1e-3)
    assert np.allclose(got[co:], (y * y).sum(0), rtol=1e-5, atol=1e-3)
    gemm(d, xd, wd, None, out)
    again = np.frombuffer(cs.get((4 * co,)).tobytes(), np.float64)
    assert np.array_equal(got, again)


SMALL_C = [c for c in CONVS if c[3] % 32 != 0 and c[5] > 1]


@pytest.mark.parametrize("shape", SMALL_C)
@pytest.mark.parametrize("kind", [CONV_FWD, CONV_WGRAD])
def test_manual_a_route(shape, kind):
    """Builder-warp gather route (no im2col) for channels % 32 != 0."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    K.nncb_gemm_set_manual_a(1)
    try:
        if kind == CONV_FWD:
            tc, ex = run_both(kind, g, Dev(x), Dev(w), None, (n, g["oh"], g["ow"], co), expect_tc=True)
        else:
            tc, ex = run_both(kind, g, Dev(x), Dev(gy), None, (k, k, ci, co), expect_tc=True)
    finally:
        K.nncb_gemm_set_manual_a(0)
    check(tc, ex)


PAIR_CONVS = [c for c in CONVS if c[3] % 32 == 0 or c[5] == 1] + [(2, 30, 30, 64, 256, 3, 1), (3, 20, 20, 128, 64, 3, 2)]


@pytest.mark.parametrize("shape", PAIR_CONVS)
@pytest.mark.parametrize("tile", [0x10000 | 128, 0x10000 | 256])
def test_cta_pair(shape, tile):
    """CTA pairs (tcgen05 cta_group::2, 256-row tiles over two SMs, each CTA
    staging half of B) for the three convolution contractions."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    K.nncb_gemm_force_tile(tile)
    try:
        tc, ex = run_both(CONV_FWD, g, Dev(x), Dev(w), None, (n, g["oh"], g["ow"], co), expect_tc=True)
        check(tc, ex)
        if (k == 1 or (ci % 32 == 0 and co % 32 == 0)) and s <= 2:
            tc, ex = run_both(CONV_DGRAD, g, Dev(gy), Dev(w), None, (n, ih, iw, ci), expect_tc=True)
            check(tc, ex)
        tc, ex = run_both(CONV_WGRAD, g, Dev(x), Dev(gy), None, (k, k, ci, co), expect_tc=True)
        check(tc, ex)
    finally:
        K.nncb_gemm_force_tile(0)


@pytest.mark.parametrize("tile", [0x10000 | 128, 0x10000 | 256])
@pytest.mark.parametrize("b,i,o", [(300, 256, 320), (1024, 512, 512), (64, 96, 160)])
def test_cta_pair_dense(b, i, o, tile):
    """CTA pairs on the dense contractions (1x1 convolutions over [batch, 1, 1, features])."""
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (b, i)).astype(np.float32)
    w = rng.uniform(-1, 1, (i, o)).astype(np.float32)
    bias = rng.uniform(-1, 1, o).astype(np.float32)
    gy = rng.uniform(-1, 1, (b, o)).astype(np.float32)
    geo = dict(batch=b, in_f=i, out_f=o)
    K.nncb_gemm_force_tile(tile)
    try:
        for kind, args, shape in [(DENSE_FWD, (Dev(x), Dev(w), Dev(bias)), (b, o)),
                                  (DENSE_DGRAD, (Dev(gy), Dev(w), None), (b, i)),
                                  (DENSE_WGRAD, (Dev(x), Dev(gy), None), (i, o))]:
            tc, ex = run_both(kind, geo, *args, shape, expect_tc=True)
            check(tc, ex)
    finally:
        K.nncb_gemm_force_tile(0)


@pytest.mark.parametrize("tile", [0x40000 | 128, 0x40000 | 256, 0x50000 | 256, 0x60000 | 128])
@pytest.mark.parametrize("shape", [(2, 14, 14, 64, 64, 3, 1), (2, 13, 11, 64, 96, 3, 2), (4, 7, 7, 128, 256, 1, 1),
                                   (3, 8, 8, 96, 128, 3, 1)])
def test_conv_fwd_transposed_weights(shape, tile):
    """Forward convolution with the weights transposed to K-major on the fly
    (autotune bit 18), alone and with CTA pairs / wide staging."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    bias = rng.uniform(-1, 1, co).astype(np.float32)
    K.nncb_gemm_force_tile(tile)
    try:
        tc, ex = run_both(CONV_FWD, g, Dev(x), Dev(w), Dev(bias), (n, g["oh"], g["ow"], co), expect_tc=True)
        check(tc, ex)
        geo = dict(batch=37, in_f=ci, out_f=co)
        xd = rng.uniform(-1, 1, (37, ci)).astype(np.float32)
        wd = rng.uniform(-1, 1, (ci, co)).astype(np.float32)
        tc, ex = run_both(DENSE_FWD, geo, Dev(xd), Dev(wd), Dev(bias), (37, co), expect_tc=True)
        check(tc, ex)
    finally:
        K.nncb_gemm_force_tile(0)


@pytest.mark.parametrize("res", [False, True])
@pytest.mark.parametrize("shape,tile", [((2, 14, 14, 64, 64, 3, 1), 0), ((4, 7, 7, 128, 256, 1, 1), 0),
                                        ((2, 13, 11, 64, 96, 3, 2), 0), ((3, 8, 8, 96, 128, 3, 1), 0x10000 | 256),
                                        ((2, 16, 16, 64, 32, 1, 1), 0), ((16, 56, 56, 64, 64, 1, 1), 0),
                                        ((4, 28, 28, 256, 64, 1, 1), 256), ((8, 14, 14, 256, 128, 3, 1), 0x10000 | 256)])
def test_dgrad_relu_grad_epilogue(shape, tile, res):
    """Dgrad epilogue that emits the gradient at the input of the following
    ReLU (dy = mask > 0 ? acc (+ residual) : 0) with the BatchNorm backward sums
    of dy (NNCB_EPI_RELU_GRAD), against the exact dgrad + numpy."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(21)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    mask = np.maximum(rng.uniform(-1, 1, (n, ih, iw, ci)), 0).astype(np.float32)
    resid = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32) if res else None
    x = rng.uniform(-2, 2, (n, ih, iw, ci)).astype(np.float32)
    stats = np.concatenate([rng.uniform(-0.5, 0.5, ci), rng.uniform(0.5, 2, ci)]).astype(np.float32)
    gyd, wd = Dev(gy), Dev(w)
    ex = Dev(nbytes=mask.nbytes)
    gemm(GemmDesc(kind=CONV_DGRAD, precision=1, epilogue=0, **g), gyd, wd, None, ex)
    exact = ex.get(mask.shape).astype(np.float64)
    md, xd, sd = Dev(mask), Dev(x), Dev(stats)
    rd = Dev(resid) if res else None
    sums, out = Dev(nbytes=2 * ci * 8), Dev(nbytes=mask.nbytes)
    d = GemmDesc(kind=CONV_DGRAD, precision=0, epilogue=8, **g)
    d.eg_mask, d.eg_x, d.eg_stats, d.eg_sums = md.p, xd.p, sd.p, sums.p
    d.eg_res = rd.p if res else None
    K.nncb_gemm_force_tile(tile)
    try:
        gemm(d, gyd, wd, None, out)
        assert K.nncb_gemm_last_path() == 1
    finally:
        K.nncb_gemm_force_tile(0)
    want = np.where(mask > 0, exact + (resid if res else 0), 0.0)
    got = out.get(mask.shape)
    assert np.max(np.abs(got - want)) <= 2e-2 * np.max(np.abs(want))
    raw = np.empty(2 * ci, np.float64)
    assert K.nncb_d2h(ctx(), raw.ctypes.data, sums.p, raw.nbytes) == 0
    K.nncb_sync(ctx())
    xhat = (x.astype(np.float64) - stats[:ci]) * stats[ci:]
    s1 = want.reshape(-1, ci).sum(0)
    s2 = (want * xhat).reshape(-1, ci).sum(0)
    assert np.linalg.norm(raw[:ci] - s1) <= 2e-2 * np.linalg.norm(s1)
    assert np.linalg.norm(raw[ci:] - s2) <= 2e-2 * np.linalg.norm(s2)


@pytest.mark.parametrize("shape", [(2, 32, 32, 3, 64, 7, 2), (2, 17, 23, 3, 32, 7, 2)])
def test_s2d_wgrad_reuses_forward_lowering(shape):
    """NNCB_EPI_A_UNCHANGED: a weight gradient after the forward conv on the
    same activation reuses the forward's space-to-depth input (one lowering
    launch fewer) and matches the exact wgrad; the hint on a different tensor
    re-lowers (still correct)."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    x2 = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    xd, x2d, wd, gyd = Dev(x), Dev(x2), Dev(w), Dev(gy)
    y = Dev(nbytes=gy.nbytes)
    dw = Dev(nbytes=w.nbytes)
    gemm(GemmDesc(kind=CONV_WGRAD, precision=0, epilogue=16, **g), xd, gyd, None, dw)   # autotune outside the count
    for xs, other in ((xd, None), (x2d, xd)):
        ex = Dev(nbytes=w.nbytes)
        gemm(GemmDesc(kind=CONV_WGRAD, precision=1, epilogue=0, **g), xs, gyd, None, ex)
        gemm(GemmDesc(kind=CONV_FWD, precision=0, epilogue=0, **g), other or xs, wd, None, y)
        before = K.nncb_launch_count(ctx())
        dw = Dev(nbytes=w.nbytes)
        gemm(GemmDesc(kind=CONV_WGRAD, precision=0, epilogue=16, **g), xs, gyd, None, dw)
        launched = K.nncb_launch_count(ctx()) - before
        assert K.nncb_gemm_last_path() == 1
        check(dw.get(w.shape), ex.get(w.shape).astype(np.float64))
        if other is None:
            # reuse: no space-to-depth input launch (GEMM + weight fold-back [+ split-K reduce])
            assert launched <= 3, launched


def test_transpose_batch_bitwise():
    """nncb_transpose_batch: several row-major matrices (ragged sizes) into
    their transposes in one launch, bit for bit."""
    from tests.nncb_ctypes import TransposeJob
    rng = np.random.default_rng(12)
    shapes = [(576, 64), (33, 70), (1, 5), (2304, 256), (147, 64)]
    mats = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    src = [Dev(m) for m in mats]
    dst = [Dev(nbytes=m.nbytes) for m in mats]
    jobs, t0 = [], 0
    for m, s, d in zip(mats, src, dst):
        jobs.append(TransposeJob(s.p, d.p, m.shape[0], m.shape[1], t0))
        t0 += -(-m.shape[0] // 32) * -(-m.shape[1] // 32)
    table = (TransposeJob * len(jobs))(*jobs)
    jd = Dev(nbytes=ctypes.sizeof(table))
    assert K.nncb_h2d(ctx(), jd.p, ctypes.addressof(table), ctypes.sizeof(table)) == 0
    assert K.nncb_transpose_batch(ctx(), jd.p, len(jobs), t0) == 0
    for m, d in zip(mats, dst):
        assert np.array_equal(d.get((m.shape[1], m.shape[0])), m.T)


@pytest.mark.parametrize("shape", [(2, 14, 14, 64, 64, 3, 1), (4, 7, 7, 128, 256, 1, 1), (2, 13, 11, 64, 96, 3, 2)])
def test_conv_fwd_caller_kmajor_weights(shape):
    """b_kmajor: a forward conv reading the caller's K-major weight copy (the
    K-major tile forced) matches the exact path."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(13)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    xd, wd, wk = Dev(x), Dev(w), Dev(np.ascontiguousarray(w.reshape(-1, co).T))
    ex = Dev(nbytes=n * g["oh"] * g["ow"] * co * 4)
    gemm(GemmDesc(kind=CONV_FWD, precision=1, epilogue=0, **g), xd, wd, None, ex)
    out = Dev(nbytes=n * g["oh"] * g["ow"] * co * 4)
    d = GemmDesc(kind=CONV_FWD, precision=0, epilogue=0, **g)
    d.b_kmajor = wk.p
    K.nncb_gemm_force_tile(0x40000 | 128)
    try:
        before = K.nncb_launch_count(ctx())
        gemm(d, xd, wd, None, out)
        assert K.nncb_gemm_last_path() == 1
        assert K.nncb_launch_count(ctx()) - before == 1   # no per-call transpose
    finally:
        K.nncb_gemm_force_tile(0)
    check(out.get((n, g["oh"], g["ow"], co)), ex.get((n, g["oh"], g["ow"], co)).astype(np.float64))


HALO_CONVS = [(2, 14, 14, 64, 64, 3, 1), (2, 56, 56, 64, 64, 3, 1), (1, 28, 28, 128, 128, 3, 1),
              (3, 9, 13, 32, 64, 3, 1), (2, 30, 30, 256, 256, 3, 1)]


@pytest.mark.parametrize("shape", HALO_CONVS)
@pytest.mark.parametrize("tile", [0x80000 | 64, 0x80000 | 128, 0x80000 | 0x40000 | 128, 0x80000 | 256, 0x180000 | 64,
                                  0x180000 | 0x40000 | 64, 0x280000 | 64, 0x280000 | 0x40000 | 64])
def test_conv_fwd_halo(shape, tile):
    """3x3 stride-1 forward through halo patches (one (TW+2) x TH patch per
    channel block and kernel row, taps as shifted descriptors), with bias and
    BatchNorm column statistics, against the exact path."""
    n, ih, iw, ci, co, k, s = shape
    if (tile & 0xffff) > 64 and co <= 64 and (tile & 0xffff) == 256:
        pytest.skip("256-wide tile on a 64-channel output")
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(17)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    bias = rng.uniform(-1, 1, co).astype(np.float32)
    xd, wd, bd = Dev(x), Dev(w), Dev(bias)
    oshape = (n, g["oh"], g["ow"], co)
    ex = Dev(nbytes=int(np.prod(oshape)) * 4)
    gemm(GemmDesc(kind=CONV_FWD, precision=1, epilogue=1, **g), xd, wd, bd, ex)
    out = Dev(nbytes=int(np.prod(oshape)) * 4)
    cs = Dev(nbytes=2 * co * 8)
    d = GemmDesc(kind=CONV_FWD, precision=0, epilogue=1 | 4, **g)
    d.colstats = cs.p
    K.nncb_gemm_force_tile(tile)
    try:
        gemm(d, xd, wd, bd, out)
        assert K.nncb_gemm_last_path() == 1
    finally:
        K.nncb_gemm_force_tile(0)
    want = ex.get(oshape).astype(np.float64)
    check(out.get(oshape), want)
    raw = np.empty(2 * co, np.float64)
    assert K.nncb_d2h(ctx(), raw.ctypes.data, cs.p, raw.nbytes) == 0
    K.nncb_sync(ctx())
    s1 = want.reshape(-1, co).sum(0)
    s2 = (want ** 2).reshape(-1, co).sum(0)
    assert np.linalg.norm(raw[:co] - s1) <= 2e-2 * np.linalg.norm(s1)
    assert np.linalg.norm(raw[co:] - s2) <= 2e-2 * np.linalg.norm(s2)


@pytest.mark.parametrize("shape", HALO_CONVS[:4])
@pytest.mark.parametrize("tile", [0x80000 | 64, 0x80000 | 128, 0x180000 | 64, 0x280000 | 64])
def test_conv_dgrad_halo(shape, tile):
    """3x3 stride-1 input gradient through halo patches of dY against the
    exact dgrad."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    rng = np.random.default_rng(19)
    gy = rng.uniform(-1, 1, (n, g["oh"], g["ow"], co)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    gyd, wd = Dev(gy), Dev(w)
    ex, out = Dev(nbytes=n * ih * iw * ci * 4), Dev(nbytes=n * ih * iw * ci * 4)
    gemm(GemmDesc(kind=CONV_DGRAD, precision=1, epilogue=0, **g), gyd, wd, None, ex)
    K.nncb_gemm_force_tile(tile)
    try:
        gemm(GemmDesc(kind=CONV_DGRAD, precision=0, epilogue=0, **g), gyd, wd, None, out)
        assert K.nncb_gemm_last_path() == 1
    finally:
        K.nncb_gemm_force_tile(0)
    check(out.get((n, ih, iw, ci)), ex.get((n, ih, iw, ci)).astype(np.float64))


def test_dgrad_halo_relu_grad_epilogue():
    """A forced halo tile with the relu-grad epilogue falls back to the regular
    tile (halo launches have no side-tile build) and stays correct."""
    test_dgrad_relu_grad_epilogue((2, 14, 14, 64, 64, 3, 1), 0x80000 | 64, True)


@pytest.mark.parametrize("shape", [(2, 32, 32, 3, 64, 7, 2), (2, 17, 23, 3, 32, 7, 2), (4, 64, 64, 3, 64, 7, 2)])
@pytest.mark.parametrize("tile", [0x80000 | 64, 0x80000 | 0x40000 | 64, 0x280000 | 64, 0x280000 | 0x40000 | 64])
def test_stem_space_to_depth_halo(shape, tile):
    """The space-to-depth stem's lowered conv (4 kernel rows x 2 taps spaced 2)
    through halo patches, against the exact path (bit 21: its eight B tiles
    resident in shared memory)."""
    n, ih, iw, ci, co, k, s = shape
    g = conv_geom(n, ih, iw, ci, co, k, s)
    if g["ow"] < 8:
        pytest.skip("output narrower than a halo tile")
    rng = np.random.default_rng(23)
    x = rng.uniform(-1, 1, (n, ih, iw, ci)).astype(np.float32)
    w = rng.uniform(-1, 1, (k, k, ci, co)).astype(np.float32)
    xd, wd = Dev(x), Dev(w)
    oshape = (n, g["oh"], g["ow"], co)
    ex, out = Dev(nbytes=int(np.prod(oshape)) * 4), Dev(nbytes=int(np.prod(oshape)) * 4)
    gemm(GemmDesc(kind=CONV_FWD, precision=1, epilogue=0, **g), xd, wd, None, ex)
    K.nncb_gemm_force_tile(tile)
    try:
        gemm(GemmDesc(kind=CONV_FWD, precision=0, epilogue=0, **g), xd, wd, None, out)
        assert K.nncb_gemm_last_path() == 1
    finally:
        K.nncb_gemm_force_tile(0)
    check(out.get(oshape), ex.get(oshape).astype(np.float64))
