"""Softmax cross-entropy loss (extension: north star "softmax-loss layers"; the
reference has only L1, runtime.cpp:468-483) -- the device kernel against the
float64 restatement (oracle/restated64.softmax_ce, itself pinned to torch f64
and to finite differences in tests/test_oracle64.py), and a C1 training step
with it, launch by launch and end to end."""
import ctypes

import numpy as np
import pytest

import paper_2205_10357_b200 as P
from oracle import restated64 as R64
from paper_2205_10357_b200 import workloads as W
from tests.nncb_ctypes import K, Dev, ctx

pytestmark = pytest.mark.gpu
K.nncb_softmax_ce.restype = ctypes.c_int
K.nncb_softmax_ce.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int64]


def ok(rc):
    assert rc == 0, K.nncb_last_error().decode()
    assert K.nncb_sync(ctx()) == 0


@pytest.mark.parametrize("rows,C", [(256, 1000), (3, 10), (1, 1), (7, 4099)])
def test_softmax_ce_kernel_vs_f64(rows, C):
    rng = np.random.default_rng(rows * 7 + C)
    z = rng.normal(0, 3, (rows, C)).astype(np.float32)
    z[0, :] += 80.0                      # a large-magnitude row: the max shift keeps exp finite
    t = rng.uniform(0, 1, (rows, C)).astype(np.float32)
    t /= t.sum(axis=1, keepdims=True)
    zd, td, gd, ld = Dev(z), Dev(t), Dev(nbytes=z.nbytes), Dev(nbytes=8)
    ok(K.nncb_softmax_ce(ctx(), zd.p, td.p, gd.p, ld.p, rows, C))
    loss = np.frombuffer(ld.get((2,)).tobytes(), np.float64)[0]
    ol, og = R64.softmax_ce(z.astype(np.float64), t.astype(np.float64))
    assert abs(loss - ol) <= 1e-12 * max(1.0, abs(ol))
    g = gd.get(z.shape).astype(np.float64)
    assert np.max(np.abs(g - og)) <= 1e-6 * max(np.max(np.abs(og)), 1e-30)   # fp32 rounding of each entry
    # deterministic: a second launch is bitwise identical
    gd2, ld2 = Dev(nbytes=z.nbytes), Dev(nbytes=8)
    ok(K.nncb_softmax_ce(ctx(), zd.p, td.p, gd2.p, ld2.p, rows, C))
    assert np.array_equal(gd.get(z.shape), gd2.get(z.shape)) and ld.get((2,)).tobytes() == ld2.get((2,)).tobytes()


def _targets(rows, C, seed):
    rng = np.random.default_rng(seed)
    t = rng.uniform(0, 1, (rows, C))
    return (t / t.sum(axis=1, keepdims=True)).astype(np.float32)


def test_c1_softmax_ce_fp32_step_vs_f64():
    """Exact-fp32 GEMM mode: the whole C1 (no BN) step with the softmax loss
    against the float64 truth at 1e-5 (north star fp32 tolerance)."""
    doc = W.c1_small_cnn(16, bn=False)
    x = W.uniform((16, 32, 32, 3), 1, "x")
    t = _targets(16, 10, 3)
    m = P.CompiledModel(doc, precision=P.PREC_FP32, loss="softmax_ce")
    o = R64.F64Model(doc, {w: m.weight(w) for w in m.weight_shapes})
    loss, grads = m.gradients({"x": x}, t)
    oloss, ograds = o.gradients({"x": x}, t, loss="softmax_ce")
    assert abs(loss - oloss) <= 1e-6 * abs(oloss)
    for w, g in ograds.items():
        err = np.linalg.norm(grads[w] - g) / np.linalg.norm(g)
        assert err < 1e-5, (w, err)


def test_c1_bn_softmax_ce_tf32_step():
    doc = W.c1_small_cnn(32, bn=True)
    x = W.uniform((32, 32, 32, 3), 1, "x")
    t = _targets(32, 10, 4)
    m = P.CompiledModel(doc, precision=P.PREC_TF32, loss="softmax_ce")
    weights = {w: m.weight(w) for w in m.weight_shapes}
    fwd = m.run({"x": x}, role="train_fwd", outputs=["p1.argmax", "p2.argmax"])
    am = {p: fwd[p + ".argmax"] for p in ("p1", "p2")}
    loss, grads = m.gradients({"x": x}, t)
    for emulate in ("tf32", None):
        o = R64.F64Model(doc, weights, emulate=emulate)
        oloss, ograds = o.gradients({"x": x}, t, loss="softmax_ce", argmax=am)
        assert abs(loss - oloss) <= 2e-2 * abs(oloss)
        scale = max(np.linalg.norm(g) for g in ograds.values())
        for w, g in ograds.items():
            if np.linalg.norm(g) < 1e-6 * scale:   # conv bias ahead of BatchNorm
                continue
            err = np.linalg.norm(grads[w] - g) / np.linalg.norm(g)
            assert err < 2e-2, (emulate, w, err)
    # five SGD steps follow the float64 oracle's trajectory (each step's loss
    # within 2e-2; the update itself is the bit-exact SGD kernel)
    o = R64.F64Model(doc, {w: m.weight(w) for w in m.weight_shapes})
    for _ in range(5):
        loss = m.train_step({"x": x}, t, 0.01)
        oloss, og = o.gradients({"x": x}, t, loss="softmax_ce")
        for k, v in og.items():
            o.w[k] = o.w[k] - 0.01 * v
        assert abs(loss - oloss) <= 2e-2 * abs(oloss), (loss, oloss)
