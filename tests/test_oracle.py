"""Pins the oracle before anything is checked against it (CPU only).

1. The reference itself (compiled from /root/reference sources) passes its own
   acceptance suite AC-1..AC-10 (tests/acceptance.cpp).
2. The C restatement (oracle/nnc_oracle.c) reproduces the reference's hand-
   computed known answers and is BIT-EXACT against the reference on the C1
   graph (forward values and every weight gradient), via the committed golden
   fixture generated from the reference (tests/golden/make_golden.py).
3. The restated initializer equals the reference InitStream.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import restated as O
from paper_2205_10357_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ACCEPTANCE = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "acceptance")


@pytest.fixture(scope="module")
def known():
    with open(os.path.join(GOLD, "known_answers.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def c1():
    return dict(np.load(os.path.join(GOLD, "c1_ref.npz")))


needs_oracle = pytest.mark.skipif(not O.available(), reason="oracle/_ref/libnnc_oracle.so not built")


@pytest.mark.skipif(not (os.path.exists(ACCEPTANCE) and os.path.isdir("/root/reference/proj/tests")),
                    reason="reference acceptance binary / sources not present")
def test_reference_acceptance_suite():
    r = subprocess.run([ACCEPTANCE], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 10


@needs_oracle
def test_known_answers_restated(known):
    import ctypes
    L = O.lib()
    # dense toy (test_autodiff.cpp:44-73)
    k = known["dense_toy"]
    x = np.array([k["x"]], np.float32)
    w = np.array(k["W"], np.float32)
    b = np.array(k["b"], np.float32)
    y = np.zeros((1, 2), np.float32)
    L.o_dense(O._f(x), O._f(w), O._f(b), O._f(y), O.I64(1), O.I64(2), O.I64(2))
    assert y.tolist() == [k["y"]]
    g = np.array([k["upstream"]], np.float32)
    gw = np.zeros((2, 2), np.float32)
    L.o_dense_grad_weight(O._f(x), O._f(g), O._f(gw), O.I64(1), O.I64(2), O.I64(2))
    assert gw.tolist() == k["gW"]
    gb = np.zeros(2, np.float32)
    L.o_sum_cols(O._f(g), O._f(gb), O.I64(1), O.I64(2))
    assert gb.tolist() == k["gb"]
    gx = np.zeros((1, 2), np.float32)
    L.o_dense_grad_input(O._f(g), O._f(w), O._f(gx), O.I64(1), O.I64(2), O.I64(2))
    assert gx.tolist() == [k["gx"]]
    # relu backward masks on x > 0 (test_autodiff.cpp:75-90)
    k = known["relu_backward"]
    xr, gr, out = np.array(k["x"], np.float32), np.array(k["upstream"], np.float32), np.zeros(2, np.float32)
    L.o_relu_grad(O._f(xr), O._f(gr), O._f(out), O.I64(2))
    assert out.tolist() == k["gx"]
    # maxpool tie -> first in scan order (test_autodiff.cpp:199-219)
    k = known["maxpool_tie"]
    xp = np.array(k["x"], np.float32).reshape(1, 1, 2, 1)
    pp, oshape = O.pool_params(xp.shape, tuple(k["kernel"]), (1, 1))
    yp, idx = np.zeros(oshape, np.float32), np.zeros(oshape, np.float32)
    L.o_maxpool2d(O._f(xp), O._f(yp), O._f(idx), pp)
    assert idx.ravel()[0] == k["argmax"]
    gp = np.full(oshape, k["upstream"], np.float32)
    gxp = np.zeros(xp.shape, np.float32)
    L.o_maxpool2d_grad(O._f(idx), O._f(gp), O._f(gxp), pp)
    assert gxp.ravel().tolist() == k["gx"]
    # l1 (test_runtime.cpp:67-75) and sgd (test_runtime.cpp:100-106)
    k = known["l1"]
    p, t, gl = np.array([k["p"]], np.float32), np.array([k["t"]], np.float32), np.zeros(1, np.float32)
    assert L.o_l1_loss(O._f(p), O._f(t), O._f(gl), O.I64(1)) == k["loss"]
    assert gl[0] == k["grad"]
    k = known["sgd"]
    ws, gs = np.array([k["w"]], np.float32), np.array([k["g"]], np.float32)
    L.o_sgd(O._f(ws), O._f(gs), O.I64(1), ctypes.c_double(k["lr"]))
    assert ws[0] == k["w_after"]


@needs_oracle
def test_restated_c1_bitexact_vs_reference_golden(c1):
    doc = bytes(c1["document"]).decode()
    m = O.OracleModel(doc)
    for k in c1:
        if k.startswith("w0/"):
            assert np.array_equal(m.w[k[3:]], c1[k]), "initializer " + k
    out = m.forward({"x": c1["x"]}, training=False)["fc"]
    assert np.array_equal(out, c1["fc"])
    loss, grads = m.gradients({"x": c1["x"]}, c1["target"])
    assert loss == float(c1["loss"][0])
    for k in c1:
        if k.startswith("grad/"):
            assert np.array_equal(grads[k[5:]], c1[k]), k


def test_init_stream_matches_reference(ref):
    for name, idx in [("x", 0), ("c1.weight", 5), ("fc.bias", 3)]:
        want = ref.init_uniform(7, name, idx, -1.0, 1.0)
        assert O.init_uniform(7, name, idx + 1, -1.0, 1.0)[idx] == want
        assert W.init_stream(7, name, idx + 1, -1.0, 1.0)[idx] == want


def test_reference_c1_regenerates_golden(ref, c1):
    """The committed fixture is what the reference produces right now."""
    doc = bytes(c1["document"]).decode()
    r = ref.RefModel(doc, 1)
    assert np.array_equal(r.run({"x": c1["x"]})["fc"].astype(np.float32), c1["fc"])


@needs_oracle
def test_restated_bn_gelu_ln_gradients_vs_finite_differences():
    """Extension ops (parity unpinned by the reference): the restated gradients
    agree with central finite differences of the restated forward in the
    reference's grad_check style (autodiff.cpp:325-400, loss sum|y - t|)."""
    doc = json.dumps({"dialect": "dlb", "name": "ext", "seed": 3,
                      "inputs": [{"name": "x", "dtype": "f32", "shape": [6, 8]}], "outputs": ["ln"],
                      "nodes": [{"name": "d", "op": "dense", "inputs": ["x"], "attrs": {"units": 8}},
                                {"name": "bn", "op": "batch_normalization", "inputs": ["d"]},
                                {"name": "g", "op": "gelu", "inputs": ["bn"]},
                                {"name": "ln", "op": "layer_normalization", "inputs": ["g"]}]})
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (6, 8)).astype(np.float32)
    t = rng.uniform(4, 6, (6, 8)).astype(np.float32)
    m = O.OracleModel(doc)
    m.w["bn.gamma"] = rng.uniform(0.5, 1.5, 8).astype(np.float32)
    m.w["ln.gamma"] = rng.uniform(0.5, 1.5, 8).astype(np.float32)
    _, grads = m.gradients({"x": x}, t)
    n = t.size

    def loss(w):
        saved = {k: v.copy() for k, v in m.w.items()}
        m.w.update(w)
        y = m.forward({"x": x}, training=True)["ln"].astype(np.float64)
        m.w = saved
        return np.abs(y - t).sum() / n

    h = 1e-2
    for name in ["d.weight", "bn.gamma", "bn.beta", "ln.gamma", "ln.beta"]:
        w0 = m.w[name]
        for i in range(min(w0.size, 6)):
            wp, wm = w0.copy(), w0.copy()
            wp.flat[i] += h
            wm.flat[i] -= h
            fd = (loss({name: wp}) - loss({name: wm})) / (2 * h)
            an = float(grads[name].flat[i])
            assert abs(fd - an) <= 2e-2 * max(abs(fd), abs(an), 1e-2), (name, i, fd, an)
