"""GPU model-level parity: whole training steps of the B200 path against the
committed reference golden fixture (no /root/reference needed at run time) and
against the restated oracle (oracle/restated.py) for graphs with the extension
ops the reference lacks (BatchNorm, GELU, LayerNorm).

Tolerances (north star): exact-fp32 GEMM mode -> bit-exact where the reference
has the op; extension-op graphs 1e-5 of max|oracle| forward and 1e-4 backward
(statistics are reduced in a different order, in double); tcgen05 tf32 mode
2e-2 of max|oracle|.
"""
import os

import numpy as np
import pytest

import paper_2205_10357_b200 as P
from oracle import restated as O
from paper_2205_10357_b200 import workloads as W

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(got, want):
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(np.asarray(got, np.float64) - want)) / max(np.max(np.abs(want)), 1e-30))


def rel_norm(got, want):
    """||got - want|| / ||want||: the tf32 gradient metric. L1's sign gradient turns
    reduced-precision perturbations of near-tie predictions into isolated O(1/N)
    flips, which an elementwise max bound over-weights."""
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(np.asarray(got, np.float64) - want) / max(np.linalg.norm(want), 1e-30))


def test_c1_against_reference_golden_fixture():
    g = dict(np.load(os.path.join(GOLD, "c1_ref.npz")))
    doc = bytes(g["document"]).decode()
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    assert np.array_equal(m.run({"x": g["x"]})["fc"], g["fc"])
    loss, grads = m.gradients({"x": g["x"]}, g["target"])
    assert abs(loss - g["loss"][0]) <= 1e-12
    for k in g:
        if k.startswith("grad/"):
            assert np.array_equal(grads[k[5:]], g[k]), k
    m2 = P.CompiledModel(doc, precision=P.PREC_FP32)
    assert abs(m2.train_step({"x": g["x"]}, g["target"], 0.05) - g["step_loss"][0]) <= 1e-12
    for k in g:
        if k.startswith("w1/"):
            assert np.array_equal(m2.weight(k[3:]), g[k]), k


def _randomize_norms(model, oracle, rng):
    for name, shape in model.weight_shapes.items():
        if name.endswith(".gamma") or name.endswith(".beta") or "moving" in name:
            lo, hi = (0.5, 1.5) if ("gamma" in name or "variance" in name) else (-0.5, 0.5)
            v = rng.uniform(lo, hi, shape).astype(np.float32)
            model.set_weight(name, v)
            oracle.w[name] = v


# tf32 backward bound 1e-1 (norm): max-pool argmax / ReLU-mask flips at near
# ties (two 2x2 pools over tf32-perturbed convolutions) move whole gradient
# entries (SURVEY.md §7 hard part 1); the flip rate itself (<1%) is asserted
# separately, and the exact-fp32 row holds the 1e-4 bound.
@pytest.mark.parametrize("precision,tol_f,tol_b", [(P.PREC_FP32, 1e-5, 1e-4), (P.PREC_TF32, 2e-2, 1e-1)])
def test_c1_batchnorm_vs_oracle(precision, tol_f, tol_b):
    doc = W.c1_small_cnn(8, bn=True)
    x = W.uniform((8, 32, 32, 3), 1, "x")
    # targets kept clear of the L1 kink, as the reference's grad_check does
    # (autodiff.cpp:361-367): reduced-precision GEMMs then cannot flip signs
    t = W.uniform((8, 10), 2, "t", 4.0, 6.0)
    m, o = P.CompiledModel(doc, precision=precision), O.OracleModel(doc)
    _randomize_norms(m, o, np.random.default_rng(0))
    assert rel(m.run({"x": x})["fc"], o.forward({"x": x}, training=False)["fc"]) < tol_f
    fwd = m.run({"x": x}, role="train_fwd")
    ofwd = o.forward({"x": x}, training=True)
    assert rel(fwd["fc"], ofwd["fc"]) < tol_f
    assert rel(fwd["bn1.stats"], o.saved["bn1.stats"]) < tol_f
    flips = np.mean(fwd["p1.argmax"] != o.saved["p1.argmax"])
    assert flips == 0 if precision == P.PREC_FP32 else flips < 0.01, flips
    loss, grads = m.gradients({"x": x}, t)
    oloss, ograds = o.gradients({"x": x}, t)
    assert abs(loss - oloss) <= tol_f * abs(oloss)
    metric = rel if precision == P.PREC_FP32 else rel_norm
    for w, g in ograds.items():
        if w in ("c1.bias", "c2.bias"):
            # a conv bias feeding BatchNorm has an analytically zero gradient (BN
            # removes the per-channel mean); both sides are rounding noise ~1e-9
            assert np.max(np.abs(grads[w])) < 1e-4 and np.max(np.abs(g)) < 1e-4, w
            continue
        assert metric(grads[w], g) < tol_b, w


@pytest.mark.parametrize("precision,tol", [(P.PREC_FP32, 1e-4), (P.PREC_TF32, 2e-2)])
def test_mlp_gelu_layernorm_vs_oracle(precision, tol):
    doc = W.mlp(64, 128, 3)
    x = W.uniform((64, 128), 1, "x")
    t = W.uniform((64, 128), 2, "t", 4.0, 6.0)
    m, o = P.CompiledModel(doc, precision=precision), O.OracleModel(doc)
    _randomize_norms(m, o, np.random.default_rng(1))
    assert rel(m.run({"x": x})["ln2"], o.forward({"x": x}, training=False)["ln2"]) < tol
    loss, grads = m.gradients({"x": x}, t)
    oloss, ograds = o.gradients({"x": x}, t)
    assert abs(loss - oloss) <= tol * abs(oloss)
    metric = rel if precision == P.PREC_FP32 else rel_norm
    for w, g in ograds.items():
        assert metric(grads[w], g) < tol, w


def test_resnet50_shaped_vs_oracle():
    """The full ResNet-50-shaped graph (BatchNorm, stem 7x7/2, strided bottlenecks,
    residual adds, global pool, dense) at a CPU-affordable size: exact-fp32 GEMM
    mode for the training step (1e-3: 53 chained batch statistics over 4 images),
    tcgen05 tf32 mode for inference (2e-2)."""
    doc = W.resnet50(4, bn=True, image=32, classes=16)
    x = W.uniform((4, 32, 32, 3), 1, "x")
    t = W.uniform((4, 16), 2, "t", 0.0, 1.0)
    o = O.OracleModel(doc)
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    _randomize_norms(m, o, np.random.default_rng(2))
    loss, grads = m.gradients({"x": x}, t)
    oloss, ograds = o.gradients({"x": x}, t)
    assert abs(loss - oloss) <= 1e-3 * abs(oloss)
    bad = {w: rel(grads[w], g) for w, g in ograds.items() if rel(grads[w], g) >= 1e-3}
    assert not bad, bad
    mt = P.CompiledModel(doc, precision=P.PREC_TF32)
    for k, v in o.w.items():
        mt.set_weight(k, v)
    assert rel(mt.run({"x": x})["fc"], o.forward({"x": x}, training=False)["fc"]) < 2e-2


def test_training_loop_like_reference_test_runtime():
    """test_runtime.cpp:242-287: dense(1->1) from w = 0, x = [1, 1], target
    [2.005, 1.995], L1 at lr 0.1 converges below 0.01 in 100 steps with >= 90
    non-increasing losses; lr = 0 repeats the loss exactly; the returned loss
    equals l1 of an inference run at the pre-step weights."""
    import json
    doc = json.dumps({"dialect": "dlb", "name": "dense1d", "seed": 0,
                      "inputs": [{"name": "x", "dtype": "f32", "shape": [2, 1]}], "outputs": ["fit"],
                      "nodes": [{"name": "fit", "op": "dense", "inputs": ["x"],
                                 "attrs": {"units": 1, "use_bias": False}}]})
    x = np.array([[1.0], [1.0]], np.float32)
    t = np.array([[2.005], [1.995]], np.float32)
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    m.set_weight("fit.weight", np.zeros((1, 1), np.float32))
    losses = [m.train_step({"x": x}, t, 0.1) for _ in range(100)]
    assert losses[-1] < 0.01
    assert sum(b <= a for a, b in zip(losses, losses[1:])) >= 90
    f = P.CompiledModel(doc, precision=P.PREC_FP32)
    f.set_weight("fit.weight", np.zeros((1, 1), np.float32))
    assert f.train_step({"x": x}, t, 0.0) == f.train_step({"x": x}, t, 0.0)
    s = P.CompiledModel(doc, precision=P.PREC_FP32)
    s.set_weight("fit.weight", np.full((1, 1), 0.37, np.float32))
    out = s.run({"x": x})["fit"].astype(np.float64)
    external = float(np.mean(np.abs(out - t.astype(np.float64))))
    assert s.train_step({"x": x}, t, 0.1) == external
    assert abs(float(s.weight("fit.weight")[0, 0]) - np.float32(0.37 + 0.1)) < 1e-7
