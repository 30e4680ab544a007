"""Pins the float64 restatement (oracle/restated64.py) before the GPU parity
tests measure the tf32 path against it (CPU only).

* Reference-vocabulary graphs (no BatchNorm): the reference itself, run in
  float64 (its runtime is dtype-generic, runtime.cpp:425-434), on the same
  weights -- losses and every weight gradient agree to ~1e-12.
* Extension ops (BatchNorm, GELU, LayerNorm, softmax cross-entropy), which the
  reference does not have: an independent implementation, torch.nn.functional
  in float64, evaluated on the same DLB document; and central finite
  differences in the reference's grad_check style (autodiff.cpp:325-400).
* The float32 C restatement (oracle/nnc_oracle.c) agrees with it to float32
  rounding on the BatchNorm graphs.
"""
import json

import numpy as np
import pytest

from oracle import restated as O
from oracle import restated64 as R64
from paper_2205_10357_b200 import workloads as W


def as_f64_doc(doc: str) -> str:
    d = json.loads(doc)
    for i in d["inputs"]:
        i["dtype"] = "f64"
    return json.dumps(d)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name,doc,xshape", [
    ("c1", lambda: W.c1_small_cnn(3, bn=False), (3, 32, 32, 3)),
    ("resnet50_s", lambda: W.resnet50(2, bn=False, image=32, classes=10), (2, 32, 32, 3)),
])
def test_f64_oracle_matches_reference_run_in_f64(ref, name, doc, xshape):
    d64 = as_f64_doc(doc())
    r = ref.RefModel(d64, 1)
    x = W.uniform(xshape, 1, "x").astype(np.float64)
    out_shape = (xshape[0], 10)
    t = W.uniform(out_shape, 2, "t", 0.0, 1.0).astype(np.float64)
    weights = {w: r.weight(w) for w in r.weight_shapes}
    m = R64.F64Model(d64, weights)
    y = m.forward({"x": x}, training=False)[m.outputs[0]]
    yr = r.run({"x": x})[m.outputs[0]]
    assert np.allclose(y, yr, rtol=1e-12, atol=1e-13)
    rloss, rgrads = r.gradients({"x": x}, t)
    loss, grads = m.gradients({"x": x}, t)
    assert abs(loss - rloss) <= 1e-12 * max(1.0, abs(rloss))
    assert set(grads) == set(rgrads)
    for w, g in rgrads.items():
        assert rel(grads[w], g) < 1e-11, (w, rel(grads[w], g))


# ---------------------------------------------------------------- torch f64
def torch_eval(doc, weights, feed, target, loss="l1"):
    """The DLB document evaluated by torch.nn.functional in float64 (NHWC data
    permuted to NCHW; TF-SAME padding spelled out; training-mode BatchNorm)."""
    import torch
    import torch.nn.functional as F
    d = json.loads(doc)
    wt = {k: torch.tensor(np.asarray(v, np.float64), requires_grad=True) for k, v in weights.items()}
    v = {k: torch.tensor(np.asarray(x, np.float64)) for k, x in feed.items()}
    for n in d["nodes"]:
        op, name, a = n["op"], n["name"], n.get("attrs", {})
        ins = [v[i] for i in n.get("inputs", [])]
        x = ins[0] if ins else None
        if op == "conv2d":
            k, s = R64._pair(a, "kernel_size"), R64._pair(a, "strides", 1)
            oh, ow, ph, pw = R64.conv_geom(tuple(x.shape), k, s, a.get("padding", "valid") == "same")
            xc = F.pad(x.permute(0, 3, 1, 2), (pw[0], pw[1], ph[0], ph[1]))
            y = F.conv2d(xc, wt[name + ".weight"].permute(3, 2, 0, 1), wt.get(name + ".bias"), stride=s)
            y = y.permute(0, 2, 3, 1)
        elif op == "dense":
            y = x @ wt[name + ".weight"]
            if name + ".bias" in wt:
                y = y + wt[name + ".bias"]
        elif op == "relu":
            y = F.relu(x)
        elif op == "gelu":
            y = F.gelu(x)
        elif op == "add":
            y = ins[0] + ins[1]
        elif op == "mul":
            y = ins[0] * ins[1]
        elif op == "flatten":
            y = x.reshape(x.shape[0], -1)
        elif op == "max_pooling2d":
            k = R64._pair(a, "pool_size")
            s = R64._pair(a, "strides") if "strides" in a else k
            y = F.max_pool2d(x.permute(0, 3, 1, 2), k, s).permute(0, 2, 3, 1)
        elif op == "global_avg_pool2d":
            y = x.mean(dim=(1, 2), keepdim=True)
        elif op == "batch_normalization":
            C = x.shape[-1]
            y = F.batch_norm(x.reshape(-1, C), None, None, wt[name + ".gamma"], wt[name + ".beta"], training=True,
                             eps=a.get("epsilon", 1e-3)).reshape(x.shape)
        elif op == "layer_normalization":
            y = F.layer_norm(x, (x.shape[-1],), wt[name + ".gamma"], wt[name + ".beta"], eps=a.get("epsilon", 1e-3))
        else:
            raise NotImplementedError(op)
        v[name] = y
    out = v[d["outputs"][0]]
    t = torch.tensor(np.asarray(target, np.float64))
    if loss == "l1":
        lv = (out - t).abs().mean()
    else:
        lv = -(t * F.log_softmax(out, dim=-1)).sum() / out.shape[0]
    lv.backward()
    return float(lv.detach()), {k: w.grad.numpy() for k, w in wt.items() if w.grad is not None}


def ext_docs():
    mlp = W.mlp(16, 32, 2)
    c1bn = W.c1_small_cnn(4, bn=True)
    rn = W.resnet50(2, bn=True, image=32, classes=10)
    return [("mlp_gelu_ln", mlp, (16, 32), (16, 32), "l1"),
            ("c1_bn", c1bn, (4, 32, 32, 3), (4, 10), "l1"),
            ("c1_bn_softmax_ce", c1bn, (4, 32, 32, 3), (4, 10), "softmax_ce"),
            ("resnet50_bn_s", rn, (2, 32, 32, 3), (2, 10), "l1")]


@pytest.mark.parametrize("name,doc,xshape,tshape,loss", ext_docs(), ids=[e[0] for e in ext_docs()])
def test_f64_oracle_extension_ops_match_torch_f64(name, doc, xshape, tshape, loss):
    pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    m = R64.F64Model(doc)
    for k in m.w:   # non-trivial affine parameters
        if k.endswith(".gamma"):
            m.w[k] = rng.uniform(0.5, 1.5, m.w[k].shape)
        if k.endswith(".beta"):
            m.w[k] = rng.uniform(-0.2, 0.2, m.w[k].shape)
    x = rng.uniform(-1, 1, xshape)
    if loss == "softmax_ce":
        t = rng.uniform(0, 1, tshape)
        t /= t.sum(axis=1, keepdims=True)
    else:
        t = rng.uniform(0, 1, tshape) + 2.0   # away from the L1 kink
    lv, grads = m.gradients({"x": x}, t, loss=loss)
    trainable = {k: v for k, v in m.w.items() if "moving" not in k}
    tl, tg = torch_eval(doc, trainable, {"x": x}, t, loss)
    assert abs(lv - tl) <= 1e-10 * max(1.0, abs(tl))
    for k, g in tg.items():
        # (a conv bias in front of a BatchNorm has an identically-zero gradient:
        # compare those on an absolute scale)
        err = np.linalg.norm(np.asarray(grads[k]) - g)
        assert err <= max(1e-9 * np.linalg.norm(g), 1e-13), (k, err, np.linalg.norm(g))


def test_f64_softmax_ce_and_bn_vs_finite_differences():
    """grad_check style (autodiff.cpp:325-400): central differences in f64, h=1e-5,
    denominator clamp 1e-8, on a dense -> BN -> GELU -> LN -> dense graph with a
    softmax cross-entropy loss."""
    doc = json.dumps({"dialect": "dlb", "name": "ext", "seed": 3,
                      "inputs": [{"name": "x", "dtype": "f64", "shape": [6, 8]}], "outputs": ["o"],
                      "nodes": [{"name": "d", "op": "dense", "inputs": ["x"], "attrs": {"units": 8}},
                                {"name": "bn", "op": "batch_normalization", "inputs": ["d"]},
                                {"name": "g", "op": "gelu", "inputs": ["bn"]},
                                {"name": "ln", "op": "layer_normalization", "inputs": ["g"]},
                                {"name": "o", "op": "dense", "inputs": ["ln"], "attrs": {"units": 5}}]})
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (6, 8))
    t = rng.uniform(0, 1, (6, 5))
    t /= t.sum(axis=1, keepdims=True)
    m = R64.F64Model(doc)
    m.w["bn.gamma"] = rng.uniform(0.5, 1.5, 8)
    m.w["ln.gamma"] = rng.uniform(0.5, 1.5, 8)
    _, grads = m.gradients({"x": x}, t, loss="softmax_ce")

    def loss():
        y = m.forward({"x": x}, training=True)["o"]
        return R64.softmax_ce(y, t)[0]

    h = 1e-5
    for name in ["d.weight", "d.bias", "bn.gamma", "bn.beta", "ln.gamma", "ln.beta", "o.weight"]:
        w0 = m.w[name]
        for i in range(min(w0.size, 8)):
            keep = w0.flat[i]
            w0.flat[i] = keep + h
            lp = loss()
            w0.flat[i] = keep - h
            lm = loss()
            w0.flat[i] = keep
            fd = (lp - lm) / (2 * h)
            an = float(grads[name].flat[i])
            assert abs(fd - an) / max(abs(fd), abs(an), 1e-8) < 1e-6 or abs(fd - an) < 1e-9, (name, i, fd, an)


@pytest.mark.skipif(not O.available(), reason="oracle/_ref/libnnc_oracle.so not built")
def test_f32_c_restatement_agrees_with_f64_on_batchnorm_graph():
    doc = W.c1_small_cnn(4, bn=True)
    x = W.uniform((4, 32, 32, 3), 1, "x")
    t = W.uniform((4, 10), 2, "t", 0.0, 1.0) + 2.0
    m32 = O.OracleModel(doc)
    m64 = R64.F64Model(doc, {k: v for k, v in m32.w.items()})
    l32, g32 = m32.gradients({"x": x}, t)
    l64, g64 = m64.gradients({"x": x}, t, argmax={k[:-7]: v for k, v in m32.saved.items() if k.endswith(".argmax")})
    assert abs(l32 - l64) <= 1e-5 * abs(l64)
    for k in g64:
        if np.linalg.norm(g64[k]) < 1e-9:   # conv bias ahead of a BatchNorm: identically zero
            assert np.linalg.norm(g32[k]) < 1e-5, k
            continue
        assert rel(g32[k], g64[k]) < 1e-4, (k, rel(g32[k], g64[k]))


def test_f64_initializer_matches_reference(ref):
    for name, idx in [("x", 0), ("c1.weight", 5), ("fc.bias", 3)]:
        assert R64.init_uniform(7, name, idx + 1, -1.0, 1.0)[idx] == ref.init_uniform(7, name, idx, -1.0, 1.0)


def _as_device(m):
    """A finished F64Model run exposed through the device_value interface."""
    def value(name):
        if name.startswith("d."):
            g = m.value_grads.get(name[2:])
            return None if g is None else g
        if name.endswith(".argmax"):
            return m.saved.get(name)
        if name.endswith(".stats"):
            st = m.saved.get(name)
            return None if st is None else np.stack([st[0], st[1]])
        return m.values.get(name)
    return value


def test_local_parity_harness_isolates_each_node():
    """oracle.restated64.local_parity re-evaluates every node from the
    "device's" own inputs: fed a tf32-emulating run, the tf32-emulating oracle
    agrees to rounding on every value, the float64 truth to the tf32 bound --
    while the end-to-end gradients of the same deep graph drift much further."""
    doc = W.resnet50(2, bn=True, image=32, classes=10)
    x = W.uniform((2, 32, 32, 3), 1, "x")
    t = W.uniform((2, 10), 2, "t", 4.0, 6.0)
    rng = np.random.default_rng(3)
    base = R64.F64Model(doc)
    w = {k: (rng.uniform(0.5, 1.5, v.shape) if k.endswith(".gamma") else v) for k, v in base.w.items()}
    dev = R64.F64Model(doc, w, emulate="tf32")
    _, dgrads = dev.gradients({"x": x}, t)
    same = R64.local_parity(R64.F64Model(doc, w, emulate="tf32"), {"x": x}, _as_device(dev), dgrads, t)
    truth = R64.local_parity(R64.F64Model(doc, w), {"x": x}, _as_device(dev), dgrads, t)
    n = sum(len(v) for v in same.values())
    assert n > 150 and len(same["weights"]) == len(dgrads)
    for part in same.values():
        assert all(e < 1e-9 for e in part.values()), part
    worst = max(max(p.values()) for p in truth.values())
    assert 1e-5 < worst < 2e-2, worst
