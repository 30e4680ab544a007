"""Kernel-level known answers and bit-exactness through the thin C-ABI (nncb.h):
the reference's hand-computed answers (tests/golden/known_answers.json) and the
restated oracle on random data, including max-pool ties."""
import ctypes
import json
import os

import numpy as np
import pytest

from oracle import restated as O
from tests.nncb_ctypes import K, Dev, ctx

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


class PoolGeom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n", "ih", "iw", "c", "kh", "kw", "sh", "sw", "oh", "ow")]


for name, args in [("nncb_maxpool_fwd", [ctypes.c_void_p, ctypes.POINTER(PoolGeom)] + [ctypes.c_void_p] * 3),
                   ("nncb_maxpool_bwd", [ctypes.c_void_p, ctypes.POINTER(PoolGeom)] + [ctypes.c_void_p] * 3),
                   ("nncb_l1_loss", [ctypes.c_void_p] * 5 + [ctypes.c_int64]),
                   ("nncb_sgd", [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double]),
                   ("nncb_bn_stats", [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
                   ("nncb_layernorm_fwd", [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
                   ("nncb_layernorm_bwd", [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
                   ("nncb_layernorm_bwd_params", [ctypes.c_void_p] * 7 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
                   ("nncb_avgpool_fwd", [ctypes.c_void_p] + [ctypes.c_int64] * 6 + [ctypes.c_void_p] * 2),
                   ("nncb_avgpool_bwd", [ctypes.c_void_p] + [ctypes.c_int64] * 6 + [ctypes.c_void_p] * 2)]:
    fn = getattr(K, name)
    fn.restype, fn.argtypes = ctypes.c_int, args


def ok(rc):
    assert rc == 0, K.nncb_last_error().decode()
    assert K.nncb_sync(ctx()) == 0


@pytest.fixture(scope="module")
def known():
    with open(os.path.join(GOLD, "known_answers.json")) as f:
        return json.load(f)


def pool(x, k, s, ties=False):
    n, ih, iw, c = x.shape
    oh, ow = (ih - k) // s + 1, (iw - k) // s + 1
    return PoolGeom(n, ih, iw, c, k, k, s, s, oh, ow), (n, oh, ow, c)


def test_maxpool_tie_and_grad_known_answer(known):
    k = known["maxpool_tie"]
    x = np.array(k["x"], np.float32).reshape(1, 1, 2, 1)
    g = PoolGeom(1, 1, 2, 1, 1, 2, 1, 1, 1, 1)
    y, idx, xd = Dev(nbytes=4), Dev(nbytes=4), Dev(x)
    ok(K.nncb_maxpool_fwd(ctx(), ctypes.byref(g), xd.p, y.p, idx.p))
    assert idx.get((1,))[0] == k["argmax"]
    gx, gy = Dev(nbytes=8), Dev(np.array([k["upstream"]], np.float32))
    ok(K.nncb_maxpool_bwd(ctx(), ctypes.byref(g), idx.p, gy.p, gx.p))
    assert gx.get((2,)).tolist() == k["gx"]


@pytest.mark.parametrize("k,s,shape", [(2, 2, (2, 9, 11, 8)), (3, 2, (2, 9, 11, 8)), (3, 1, (2, 9, 11, 8)),
                                       (3, 2, (3, 10, 12, 64)), (3, 2, (1, 16, 15, 12))])
def test_maxpool_bitexact_with_ties(k, s, shape):
    rng = np.random.default_rng(k * 10 + s)
    x = rng.integers(-3, 4, shape).astype(np.float32)   # many exact ties
    g, oshape = pool(x, k, s)
    y, idx, xd = Dev(nbytes=4 * int(np.prod(oshape))), Dev(nbytes=4 * int(np.prod(oshape))), Dev(x)
    ok(K.nncb_maxpool_fwd(ctx(), ctypes.byref(g), xd.p, y.p, idx.p))
    pp, _ = O.pool_params(x.shape, (k, k), (s, s))
    oy, oidx = np.zeros(oshape, np.float32), np.zeros(oshape, np.float32)
    O.lib().o_maxpool2d(O._f(x), O._f(oy), O._f(oidx), pp)
    assert np.array_equal(y.get(oshape), oy) and np.array_equal(idx.get(oshape), oidx)
    gy = rng.uniform(-1, 1, oshape).astype(np.float32)
    gx, gyd = Dev(nbytes=x.nbytes), Dev(gy)
    ok(K.nncb_maxpool_bwd(ctx(), ctypes.byref(g), idx.p, gyd.p, gx.p))
    ogx = np.zeros(x.shape, np.float32)
    O.lib().o_maxpool2d_grad(O._f(oidx), O._f(gy), O._f(ogx), pp)
    assert np.array_equal(gx.get(x.shape), ogx)


def test_global_avgpool_bitexact():
    x = np.random.default_rng(3).uniform(-1, 1, (3, 7, 7, 64)).astype(np.float32)
    y, xd = Dev(nbytes=3 * 64 * 4), Dev(x)
    ok(K.nncb_avgpool_fwd(ctx(), 3, 7, 7, 64, 1, 1, xd.p, y.p))
    oy = np.zeros((3, 1, 1, 64), np.float32)
    O.lib().o_avgpool(O._f(x), O._f(oy), *[O.I64(v) for v in (3, 7, 7, 64, 1, 1)])
    assert np.array_equal(y.get((3, 1, 1, 64)), oy)


@pytest.mark.parametrize("geo", [(3, 7, 7, 64, 1, 1), (2, 7, 10, 5, 3, 4), (2, 10, 9, 8, 4, 3), (1, 5, 5, 12, 5, 5),
                                 (2, 6, 6, 16, 4, 4)])
def test_adaptive_avgpool_grad_bitexact(geo):
    n, ih, iw, c, oh, ow = geo
    gy = np.random.default_rng(4).uniform(-1, 1, (n, oh, ow, c)).astype(np.float32)
    gyd, gx = Dev(gy), Dev(nbytes=n * ih * iw * c * 4)
    ok(K.nncb_avgpool_bwd(ctx(), n, ih, iw, c, oh, ow, gyd.p, gx.p))
    ogx = np.zeros((n, ih, iw, c), np.float32)
    O.lib().o_avgpool_grad(O._f(gy), O._f(ogx), *[O.I64(v) for v in geo])
    assert np.array_equal(gx.get((n, ih, iw, c)), ogx)


def test_l1_and_sgd_known_answers(known):
    k = known["l1"]
    grad, loss = Dev(nbytes=4), Dev(nbytes=8)
    pd, td = Dev(np.array([k["p"]], np.float32)), Dev(np.array([k["t"]], np.float32))
    ok(K.nncb_l1_loss(ctx(), pd.p, td.p, grad.p, loss.p, 1))
    assert grad.get((1,))[0] == k["grad"]
    assert np.frombuffer(loss.get((2,)).tobytes(), np.float64)[0] == k["loss"]
    k = known["sgd"]
    w, gd = Dev(np.array([k["w"]], np.float32)), Dev(np.array([k["g"]], np.float32))
    ok(K.nncb_sgd(ctx(), w.p, gd.p, 1, k["lr"], 1.0))
    assert w.get((1,))[0] == k["w_after"]


def test_l1_and_sgd_bitexact_random():
    rng = np.random.default_rng(5)
    p, t = rng.uniform(-2, 2, 4099).astype(np.float32), rng.uniform(-2, 2, 4099).astype(np.float32)
    t[::7] = p[::7]     # zero differences -> sign(0) = 0
    grad, loss, pd, td = Dev(nbytes=p.nbytes), Dev(nbytes=8), Dev(p), Dev(t)
    ok(K.nncb_l1_loss(ctx(), pd.p, td.p, grad.p, loss.p, p.size))
    og = np.zeros_like(p)
    ol = O.lib().o_l1_loss(O._f(p), O._f(t), O._f(og), O.I64(p.size))
    assert np.array_equal(grad.get(p.shape), og)
    assert abs(np.frombuffer(loss.get((2,)).tobytes(), np.float64)[0] - ol) <= 1e-12 * ol
    w, g = rng.uniform(-1, 1, 4099).astype(np.float32), rng.uniform(-1, 1, 4099).astype(np.float32)
    wd, gd = Dev(w), Dev(g)
    ok(K.nncb_sgd(ctx(), wd.p, gd.p, w.size, 0.0123, 1.0))
    ow = w.copy()
    O.lib().o_sgd(O._f(ow), O._f(g), O.I64(w.size), ctypes.c_double(0.0123))
    assert np.array_equal(wd.get(w.shape), ow)


def test_batchnorm_statistics_vs_oracle():
    x = np.random.default_rng(6).normal(0.3, 2.0, (4096, 96)).astype(np.float32)
    st, xd = Dev(nbytes=2 * 96 * 4), Dev(x)
    ok(K.nncb_bn_stats(ctx(), xd.p, st.p, 4096, 96, 1e-3))
    ost = np.zeros((2, 96), np.float32)
    O.lib().o_bn_stats(O._f(x), O._f(ost), O.I64(4096), O.I64(96), ctypes.c_double(1e-3))
    assert np.max(np.abs(st.get((2, 96)) - ost) / np.abs(ost)) < 1e-6


def test_layernorm_forward_vs_oracle():
    rng = np.random.default_rng(7)
    x = rng.normal(0, 1.5, (64, 4096)).astype(np.float32)
    ga, be = rng.uniform(0.5, 1.5, 4096).astype(np.float32), rng.uniform(-0.5, 0.5, 4096).astype(np.float32)
    y, xd, gd, bd = Dev(nbytes=x.nbytes), Dev(x), Dev(ga), Dev(be)
    ok(K.nncb_layernorm_fwd(ctx(), xd.p, gd.p, bd.p, y.p, 64, 4096, 1e-5))
    oy = np.zeros_like(x)
    O.lib().o_layernorm(O._f(x), O._f(ga), O._f(be), O._f(oy), O.I64(64), O.I64(4096), ctypes.c_double(1e-5))
    assert np.max(np.abs(y.get(x.shape) - oy)) / np.max(np.abs(oy)) < 1e-6


@pytest.mark.parametrize("rows,C", [(8192, 4096), (1000, 1024), (37, 256), (3, 8192), (17, 100)])
def test_layernorm_backward_with_parameter_gradients(rows, C):
    """nncb_layernorm_bwd_params: gx bitwise equal to nncb_layernorm_bwd, and
    dgamma = sum g*xhat, dbeta = sum g against the C oracle / float64 numpy
    (C=100 takes the unaligned fallback sequence)."""
    rng = np.random.default_rng(rows + C)
    x = rng.normal(0.3, 1.2, (rows, C)).astype(np.float32)
    g = rng.normal(0, 1, (rows, C)).astype(np.float32)
    ga = rng.uniform(0.5, 1.5, C).astype(np.float32)
    xd, gd, gad = Dev(x), Dev(g), Dev(ga)
    gx0, gx1 = Dev(nbytes=x.nbytes), Dev(nbytes=x.nbytes)
    dg, db = Dev(nbytes=4 * C), Dev(nbytes=4 * C)
    ok(K.nncb_layernorm_bwd(ctx(), xd.p, gad.p, gd.p, gx0.p, rows, C, 1e-5))
    ok(K.nncb_layernorm_bwd_params(ctx(), xd.p, gad.p, gd.p, gx1.p, dg.p, db.p, rows, C, 1e-5))
    assert np.array_equal(gx0.get(x.shape), gx1.get(x.shape))
    odg = np.zeros(C, np.float32)
    O.lib().o_layernorm_dgamma(O._f(x), O._f(g), O._f(odg), O.I64(rows), O.I64(C), ctypes.c_double(1e-5))
    scale = np.sqrt(rows)
    assert np.max(np.abs(dg.get((C,)) - odg)) / scale < 2e-6
    assert np.max(np.abs(db.get((C,)) - g.astype(np.float64).sum(0))) / scale < 2e-6
    # either output alone
    dg2 = Dev(nbytes=4 * C)
    ok(K.nncb_layernorm_bwd_params(ctx(), xd.p, gad.p, gd.p, gx1.p, dg2.p, None, rows, C, 1e-5))
    assert np.array_equal(dg2.get((C,)), dg.get((C,)))


@pytest.mark.parametrize("rows,C", [(4096, 64), (1000, 256), (512, 2048), (333, 128), (50, 1024)])
def test_ew_fused_bn_grad_reduce(rows, C):
    """REDUCE_BN_GRAD fused into an elementwise group: per-channel sum(g) and
    sum(g * xhat) of the value the group produces, against float64 numpy and
    the standalone nncb_bn_grad_reduce (both accumulate in double)."""
    from tests.nncb_ctypes import ew_run
    rng = np.random.default_rng(11)
    g = rng.uniform(-1, 1, (rows, C)).astype(np.float32)
    x = rng.uniform(-2, 2, (rows, C)).astype(np.float32)
    mean = x.mean(0).astype(np.float32)
    invstd = (1.0 / np.sqrt(x.var(0) + 1e-5)).astype(np.float32)
    gd, xd, md, sd = Dev(g), Dev(x), Dev(mean), Dev(invstd)
    out, sg, sgx = Dev(nbytes=g.nbytes), Dev(nbytes=C * 4), Dev(nbytes=C * 4)
    LOAD, LOAD_CH, STORE, RELU, RED = 0, 1, 2, 3, 13
    prog = [dict(op=LOAD, dst=0, slot=0), dict(op=LOAD, dst=1, slot=1), dict(op=LOAD_CH, dst=2, slot=2),
            dict(op=LOAD_CH, dst=3, slot=3), dict(op=RELU, dst=4, a=0), dict(op=STORE, a=4, slot=4),
            dict(op=RED, a=4, b=1, c=2, d=3, slot=5, e=6)]
    ew_run(prog, 5, [gd, xd, md, sd, out, sg, sgx], rows * C, C)
    gr = np.maximum(g, 0).astype(np.float64)
    xhat = (x.astype(np.float64) - mean.astype(np.float64)) * invstd.astype(np.float64)
    want_g, want_gx = gr.sum(0), (gr * xhat).sum(0)
    assert np.array_equal(out.get((rows, C)), np.maximum(g, 0))
    got_g, got_gx = sg.get((C,)), sgx.get((C,))
    scale = np.abs(gr).sum(0) + 1e-30
    assert np.max(np.abs(got_g - want_g) / scale) < 1e-6
    assert np.max(np.abs(got_gx - want_gx) / (np.abs(gr * xhat).sum(0) + 1e-30)) < 1e-6
    # same answer as the standalone reduction over the stored value
    stats = Dev(np.concatenate([mean, invstd]))
    ref_g, ref_gx = Dev(nbytes=C * 4), Dev(nbytes=C * 4)
    ok(K.nncb_bn_grad_reduce(ctx(), xd.p, stats.p, out.p, ref_g.p, ref_gx.p, rows, C))
    np.testing.assert_allclose(got_g, ref_g.get((C,)), rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(got_gx, ref_gx.get((C,)), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("rows,C", [(8192, 4096), (999, 8192), (4096, 64), (333, 2048), (7, 4)])
def test_ew_fused_column_sum(rows, C):
    """REDUCE_SUM fused into an elementwise group (the Dense bias gradient of
    the value the group stores): per-column sum in double against float64
    numpy; the stored value is unchanged."""
    from tests.nncb_ctypes import ew_run
    rng = np.random.default_rng(rows + C)
    a = rng.uniform(-1, 1, (rows, C)).astype(np.float32)
    b = rng.uniform(-1, 1, (rows, C)).astype(np.float32)
    ad, bd = Dev(a), Dev(b)
    out, s = Dev(nbytes=a.nbytes), Dev(nbytes=C * 4)
    LOAD, STORE, MUL, RSUM = 0, 2, 6, 18
    prog = [dict(op=LOAD, dst=0, slot=0), dict(op=LOAD, dst=1, slot=1), dict(op=MUL, dst=2, a=0, b=1),
            dict(op=STORE, a=2, slot=2), dict(op=RSUM, a=2, slot=3)]
    ew_run(prog, 3, [ad, bd, out, s], rows * C, C)
    prod = a * b
    assert np.array_equal(out.get((rows, C)), prod)
    want = prod.astype(np.float64).sum(0)
    scale = np.abs(prod).astype(np.float64).sum(0) + 1e-30
    assert np.max(np.abs(s.get((C,)) - want) / scale) < 1e-6


@pytest.mark.parametrize("rows,C", [(4096, 64), (1000, 256)])
def test_bn_grad_fast_matches_exact(rows, C):
    """tf32-mode BatchNorm input gradient (per-channel quotients) against the
    bit-exact form (per-element IEEE division): same operands, <= 1e-5 of max."""
    from tests.nncb_ctypes import ew_run
    rng = np.random.default_rng(12)
    x = rng.uniform(-2, 2, (rows, C)).astype(np.float32)
    g = rng.uniform(-1, 1, (rows, C)).astype(np.float32)
    mean = x.mean(0).astype(np.float32)
    inv = (1.0 / np.sqrt(x.var(0) + 1e-5)).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, C).astype(np.float32)
    xhat = (x - mean) * inv
    sg, sgx = g.sum(0).astype(np.float32), (g * xhat).sum(0).astype(np.float32)
    outs = []
    for op in (11, 14):
        slots = [Dev(x), Dev(g), Dev(mean), Dev(inv), Dev(gamma), Dev(sg), Dev(sgx), Dev(nbytes=x.nbytes)]
        prog = [dict(op=0, dst=0, slot=0), dict(op=0, dst=1, slot=1)] + \
               [dict(op=1, dst=2 + i, slot=2 + i) for i in range(5)] + \
               [dict(op=op, dst=7, a=0, b=1, c=2, d=3, e=4, f=5, h=6, imm=float(rows)), dict(op=2, a=7, slot=7)]
        ew_run(prog, 8, slots, rows * C, C)
        outs.append(slots[7].get((rows, C)))
    exact, fast = outs
    ref = gamma * inv * (g - (sg + xhat * sgx) / rows)
    assert np.max(np.abs(exact - ref)) <= 1e-5 * np.max(np.abs(ref))
    assert np.max(np.abs(fast - exact)) <= 1e-5 * np.max(np.abs(exact))


def test_ew_two_fused_bn_grad_reductions():
    """Two REDUCE_BN_GRAD in one group (the two BatchNorms of a residual join
    receive the same gradient): each matches the standalone reduction."""
    from tests.nncb_ctypes import ew_run
    rows, C = 2048, 256
    rng = np.random.default_rng(13)
    g = rng.uniform(-1, 1, (rows, C)).astype(np.float32)
    xs = [rng.uniform(-2, 2, (rows, C)).astype(np.float32) for _ in range(2)]
    stats = [(x.mean(0).astype(np.float32), (1.0 / np.sqrt(x.var(0) + 1e-5)).astype(np.float32)) for x in xs]
    gd, out = Dev(g), Dev(nbytes=g.nbytes)
    devs = [(Dev(x), Dev(m), Dev(s), Dev(nbytes=C * 4), Dev(nbytes=C * 4)) for x, (m, s) in zip(xs, stats)]
    slots = [gd, out] + [d for t in devs for d in t]
    prog = [dict(op=0, dst=0, slot=0), dict(op=3, dst=1, a=0), dict(op=2, a=1, slot=1)]
    for q in range(2):
        b = 2 + 5 * q
        r = 2 + 3 * q
        prog += [dict(op=0, dst=r, slot=b), dict(op=1, dst=r + 1, slot=b + 1), dict(op=1, dst=r + 2, slot=b + 2),
                 dict(op=13, a=1, b=r, c=r + 1, d=r + 2, slot=b + 3, e=b + 4)]
    ew_run(prog, 8, slots, rows * C, C)
    gr = np.maximum(g, 0)
    for q, (xd, md, sd, sg, sgx) in enumerate(devs):
        ref_g, ref_gx = Dev(nbytes=C * 4), Dev(nbytes=C * 4)
        st = Dev(np.concatenate(stats[q]))
        ok(K.nncb_bn_grad_reduce(ctx(), xd.p, st.p, out.p, ref_g.p, ref_gx.p, rows, C))
        np.testing.assert_allclose(sg.get((C,)), ref_g.get((C,)), rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(sgx.get((C,)), ref_gx.get((C,)), rtol=1e-5, atol=1e-5)
    assert np.array_equal(out.get((rows, C)), gr)


def test_global_avgpool_grad_signed_zero_bitwise():
    """Global pooling backward bit for bit (uint32 view), including gy = -0.0
    (0 + (-0) * scale = +0 in the reference's accumulation)."""
    n, ih, iw, c = 2, 7, 7, 2048
    gy = np.random.default_rng(9).uniform(-1, 1, (n, 1, 1, c)).astype(np.float32)
    gy.reshape(-1)[::7] = -0.0
    gy.reshape(-1)[1::7] = 0.0
    gyd, gx = Dev(gy), Dev(nbytes=n * ih * iw * c * 4)
    ok(K.nncb_avgpool_bwd(ctx(), n, ih, iw, c, 1, 1, gyd.p, gx.p))
    ogx = np.zeros((n, ih, iw, c), np.float32)
    O.lib().o_avgpool_grad(O._f(gy), O._f(ogx), *[O.I64(v) for v in (n, ih, iw, c, 1, 1)])
    assert np.array_equal(gx.get((n, ih, iw, c)).view(np.uint32), ogx.view(np.uint32))
