"""GPU parity: the B200 path (through the C-ABI) against the reference CPU
implementation compiled from /root/reference (oracle/_ref/libnncref.so) on the
same documents, weights and inputs.

Tolerances: elementwise fused groups, pooling (values + argmax indices), SGD
and the exact-fp32 GEMM mode are BIT-EXACT; the tcgen05 tf32 GEMM path is held
to 2e-2 of max|ref| (the north star's reduced-precision GEMM bound), measured
elementwise against the reference.
"""
import numpy as np
import pytest

import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W

pytestmark = pytest.mark.gpu


def rel_err(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def test_c2_chain_bitwise(ref):
    doc = W.c2_chain((4, 16, 16, 64), mode="ref")
    x = W.uniform((4, 16, 16, 64), 5, "x")
    y = W.uniform((4, 16, 16, 64), 6, "y")
    m = P.CompiledModel(doc)
    launches = [g["launches"] for g in m.describe["inference"]["groups"]]
    assert len(launches) == 1 and len(launches[0]) == 1, "depth-16 chain must be ONE fused kernel"
    got = m.run({"x": x, "y": y})
    r = ref.RefModel(doc, 0).run({"x": x, "y": y})
    (name,) = r.keys()
    assert np.array_equal(got[name], r[name].astype(np.float32))


@pytest.mark.parametrize("batch", [1, 4])
def test_c1_inference_exact(ref, batch):
    doc = W.c1_small_cnn(batch, bn=False)
    x = W.uniform((batch, 32, 32, 3), 1, "x")
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    got = m.run({"x": x})
    r = ref.RefModel(doc, 1).run({"x": x})
    assert np.array_equal(got["fc"], r["fc"].astype(np.float32))


def test_c1_inference_tf32(ref):
    doc = W.c1_small_cnn(8, bn=False)
    x = W.uniform((8, 32, 32, 3), 1, "x")
    got = P.CompiledModel(doc, precision=P.PREC_TF32).run({"x": x})
    r = ref.RefModel(doc, 1).run({"x": x})
    assert rel_err(got["fc"], r["fc"]) < 2e-2


def test_c1_train_fwd_saveset_exact(ref):
    doc = W.c1_small_cnn(2, bn=False)
    x = W.uniform((2, 32, 32, 3), 1, "x")
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    got = m.run({"x": x}, role="train_fwd")
    names = ["c1", "p1", "p1.argmax", "c2", "p2.argmax", "f", "fc"]
    r = ref.RefModel(doc, 1)
    rv = r.run({"x": x}, names=None)
    ev = r.eval_all({"x": x}, ["c1", "p1", "c2", "f", "fc"])
    for n in ["c1", "p1", "c2", "f", "fc"]:
        assert np.array_equal(got[n], ev[n].astype(np.float32)), n
    assert "p1.argmax" in got and "p2.argmax" in got


def test_c1_gradients_exact(ref):
    doc = W.c1_small_cnn(4, bn=False)
    x = W.uniform((4, 32, 32, 3), 1, "x")
    t = W.uniform((4, 10), 2, "t", 0.0, 1.0)
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    loss, grads = m.gradients({"x": x}, t)
    rloss, rgrads = ref.RefModel(doc, 1).gradients({"x": x}, t)
    assert abs(loss - rloss) <= 1e-12 * max(1.0, abs(rloss))
    for w, g in rgrads.items():
        assert np.array_equal(grads[w], g.astype(np.float32)), w


def test_c1_train_steps_match_reference(ref):
    doc = W.c1_small_cnn(4, bn=False)
    x = W.uniform((4, 32, 32, 3), 1, "x")
    t = W.uniform((4, 10), 2, "t", 0.0, 1.0)
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    r = ref.RefModel(doc, 1)
    for step in range(3):
        l1 = m.train_step({"x": x}, t, 0.05)
        l2 = r.train_step({"x": x}, t, 0.05)
        assert abs(l1 - l2) <= 1e-12 * max(1.0, abs(l2)), step
    for w in r.weight_shapes:
        assert np.array_equal(m.weight(w), r.weight(w).astype(np.float32)), w


def test_c1_gradients_tf32(ref):
    doc = W.c1_small_cnn(8, bn=False)
    x = W.uniform((8, 32, 32, 3), 1, "x")
    t = W.uniform((8, 10), 2, "t", 0.0, 1.0)
    loss, grads = P.CompiledModel(doc, precision=P.PREC_TF32).gradients({"x": x}, t)
    rloss, rgrads = ref.RefModel(doc, 1).gradients({"x": x}, t)
    assert abs(loss - rloss) <= 2e-2 * abs(rloss)
    for w, g in rgrads.items():
        assert rel_err(grads[w], g) < 2e-2, w


def test_offload_protocol_ac8():
    """The reference's offload protocol (AC-8; test_runtime.cpp:129-193,
    acceptance.cpp:511-561) on the device weight cache: the first run uploads
    every weight, a second run moves 0 weight bytes with bit-identical outputs,
    and one mutation moves exactly that weight's (64-byte aligned) bytes."""
    doc = W.c1_small_cnn(4, bn=False)
    x = W.uniform((4, 32, 32, 3), 1, "x")
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    P.sync_stats(reset=True)
    out1 = m.run({"x": x})
    s1 = P.sync_stats(reset=True)
    expect = sum(-(-int(np.prod(shape)) * 4 // 64) * 64 for shape in m.weight_shapes.values())
    assert s1["weight_bytes"] == expect
    out2 = m.run({"x": x})
    s2 = P.sync_stats(reset=True)
    assert s2["weight_bytes"] == 0
    for k in out1:
        assert np.array_equal(out1[k], out2[k]), k
    name = sorted(m.weight_shapes)[0]
    w = np.random.default_rng(3).uniform(-0.1, 0.1, m.weight_shapes[name]).astype(np.float32)
    m.set_weight(name, w)
    m.run({"x": x})
    s3 = P.sync_stats(reset=True)
    assert s3["weight_bytes"] == -(-w.size * 4 // 64) * 64


@pytest.mark.parametrize("bn", [False, True])
def test_device_memory_matches_static_estimate(bn):
    """The reference's invariant runtime high_water == estimate_peak
    (test_runtime.cpp:195-240) for the B200 bound programs: the live bytes of
    every buffer value replayed over the events equal plan::estimate_peak at the
    arena alignment, for inference and for the fused train_fwd + train_bwd
    program; the arena's address span (best-fit offsets) is reported beside it."""
    doc = W.c1_small_cnn(8, bn=bn)
    x = W.uniform((8, 32, 32, 3), 1, "x")
    t = W.uniform((8, 10), 2, "t")
    m = P.CompiledModel(doc, precision=P.PREC_FP32)
    m.run({"x": x})
    inf = m.memory("inference")
    assert inf["live_high_water"] == inf["estimate"] > 0
    assert inf["arena_bytes"] >= inf["live_high_water"] - sum(-(-int(np.prod(s)) * 4 // 256) * 256
                                                               for s in m.weight_shapes.values())
    m.trainer_prepare({"x": x}, t)
    tr = m.memory("training")
    assert tr["live_high_water"] == tr["estimate"] > 0


def test_solp_loaded_plans_execute_bitwise():
    """Deploy path: plans serialized to SOLP and loaded into a fresh model run
    bitwise-identically to the compiled ones (ref test_backends.cpp:308-333)."""
    doc = W.c1_small_cnn(8, bn=True)
    x = W.uniform((8, 32, 32, 3), 1, "x")
    t = W.uniform((8, 10), 2, "t")
    a = P.CompiledModel(doc, precision=P.PREC_FP32)
    b = P.CompiledModel(doc, precision=P.PREC_FP32)
    b.load_plans(a.save_plans())
    ra, rb = a.run({"x": x}), b.run({"x": x})
    assert ra.keys() == rb.keys() and all(np.array_equal(ra[k], rb[k]) for k in ra)
    la, ga = a.gradients({"x": x}, t)
    lb, gb = b.gradients({"x": x}, t)
    assert la == lb and all(np.array_equal(ga[k], gb[k]) for k in ga)


def test_relu_grad_epilogue_fusion_matches_separate_pass(monkeypatch):
    """Opt-in runtime pass (NNC_RELU_GRAD_EPILOGUE): the relu-grad + BatchNorm
    reduction groups move into the dgrad GEMM epilogues of a residual network
    (fewer launches per step), with the same loss and gradients as the separate
    elementwise pass to within the tf32 bound."""
    doc = W.resnet50(2, image=64)
    x = W.uniform((2, 64, 64, 3), 1, "x")
    t = W.uniform((2, 1000), 2, "t", 0.0, 1.0)
    monkeypatch.delenv("NNC_RELU_GRAD_EPILOGUE", raising=False)
    a = P.CompiledModel(doc, precision=P.PREC_TF32)
    loss_a, grads_a = a.gradients({"x": x}, t)
    a.trainer_prepare({"x": x}, t)
    n_a = len(a.profile_step(0.0))
    monkeypatch.setenv("NNC_RELU_GRAD_EPILOGUE", "1")
    b = P.CompiledModel(doc, precision=P.PREC_TF32)
    loss_b, grads_b = b.gradients({"x": x}, t)
    b.trainer_prepare({"x": x}, t)
    n_b = len(b.profile_step(0.0))
    assert n_b <= n_a - 30, (n_a, n_b)
    assert abs(loss_b - loss_a) <= 1e-3 * abs(loss_a)
    for w, g in grads_a.items():
        assert rel_err(grads_b[w], g) < 2e-2, w


def test_pipelined_train_steps_match_sequential():
    """train_steps (upload of step i+1 on the copy stream while step i runs)
    gives bitwise the same losses and weights as one train_step per batch."""
    doc = W.c1_small_cnn(8, bn=True)
    batches = [({"x": W.uniform((8, 32, 32, 3), 10 + i, "x")}, W.uniform((8, 10), 20 + i, "t")) for i in range(4)]
    a = P.CompiledModel(doc, precision=P.PREC_TF32)
    b = P.CompiledModel(doc, precision=P.PREC_TF32)
    seq = [a.train_step(x, t, 0.05) for x, t in batches]
    pipe = b.train_steps(batches, 0.05)
    assert seq == pipe
    for w in a.weight_shapes:
        assert np.array_equal(a.weight(w), b.weight(w)), w
    assert b.train_steps([], 0.05) == []
    assert len(b.train_steps(batches[:1], 0.05)) == 1


def test_pipelined_runs_match_sequential():
    """run_many (upload of run i+1 on the copy stream while run i executes)
    returns bitwise the outputs of one run() per batch, also for a subset."""
    doc = W.c1_small_cnn(8, bn=True)
    m = P.CompiledModel(doc, precision=P.PREC_TF32)
    batches = [{"x": W.uniform((8, 32, 32, 3), 30 + i, "x")} for i in range(4)]
    seq = [m.run(b) for b in batches]
    pipe = m.run_many(batches)
    assert len(pipe) == 4
    for a, b in zip(seq, pipe):
        assert a.keys() == b.keys()
        for k in a:
            assert np.array_equal(a[k], b[k]), k
    name = sorted(seq[0])[0]
    sub = m.run_many(batches[:2], outputs=[name])
    assert [list(o) for o in sub] == [[name], [name]]
    assert np.array_equal(sub[1][name], seq[1][name])
    assert m.run_many([]) == []


@pytest.mark.parametrize("precision", [P.PREC_TF32, P.PREC_BF16])
def test_bn_inference_epilogue_is_bitwise_the_separate_pass(precision, monkeypatch):
    """Inference BatchNorm + ReLU groups that only transform a forward GEMM's
    output run in that GEMM's epilogue (NNCB_EPI_BN_AFFINE | NNCB_EPI_RELU):
    the same fp32 operation sequence as the fused group's BN_INFER, so the
    outputs are bitwise those of the unfused plan, with fewer launches."""
    doc = W.resnet50(4, bn=True, image=64, classes=16)
    x = W.uniform((4, 64, 64, 3), 1, "x")
    outs, counts = [], []
    for fused in (True, False):
        if not fused:   # (read when the plan is bound, at its first run)
            monkeypatch.setenv("NNC_NO_BN_INFER_EPILOGUE", "1")
        m = P.CompiledModel(doc, precision=precision)
        rng = np.random.default_rng(9)
        for name, shape in m.weight_shapes.items():
            if "moving_variance" in name or name.endswith(".gamma"):
                m.set_weight(name, rng.uniform(0.5, 1.5, shape).astype(np.float32))
            elif "moving_mean" in name or name.endswith(".beta"):
                m.set_weight(name, rng.uniform(-0.5, 0.5, shape).astype(np.float32))
        outs.append(m.run({"x": x})["fc"])
        counts.append(len(m.profile_run({"x": x})))
        del m
    a, b = outs
    na, nb = counts
    assert np.array_equal(a, b)
    assert na <= nb - 30, (na, nb)   # the stem's and every a / b conv's BN + ReLU pass
