"""Measured layer-wise tuning on the device (backends::tune_with_report with
CUDA-event timings, reference backends.cpp:73-176): every GEMM node is timed
once per tensor-core tile candidate and the fastest is chosen; the choices
are attached to the plans, survive a SOLP round trip, and the tuned model
computes the same step as the untuned one (tile choice only changes the fp32
accumulation order)."""
import numpy as np
import pytest

import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_measured_tuning_times_tiles_and_persists_them():
    doc = W.c1_small_cnn(64, bn=True)
    m = P.CompiledModel(doc, precision=P.PREC_TF32)
    rep = m.tune(warmup=1, trials=3)
    gemm_recs = [r for r in rep["train_bwd"]["records"] + rep["train_fwd"]["records"] if r["backend"] == "b200_gemm"]
    assert gemm_recs
    by_node = {}
    for r in gemm_recs:
        by_node.setdefault(r["node"], []).append(r)
    multi = {n: rs for n, rs in by_node.items() if len(rs) > 1}
    assert multi, "no GEMM node had more than one tile candidate"
    for n, rs in by_node.items():
        chosen = [r for r in rs if r["chosen"]]
        assert len(chosen) == 1, n
        assert chosen[0]["cost_us"] == min(r["cost_us"] for r in rs)
        assert all(r["cost_us"] > 0 for r in rs)
    assert rep["attached_launches"] > 0
    tiles = {L["label"]: L["tile"] for role in ("train_fwd", "train_bwd")
             for g in m.describe[role]["groups"] for L in g["launches"] if L["kind"] == "gemm"}
    assert any(t != 0 for t in tiles.values())
    # the choices travel with the plans (SOLP)
    blob = m.save_plans()
    m2 = P.CompiledModel(doc, precision=P.PREC_TF32)
    m2.load_plans(blob)
    tiles2 = {L["label"]: L["tile"] for role in ("train_fwd", "train_bwd")
              for g in m2.describe[role]["groups"] for L in g["launches"] if L["kind"] == "gemm"}
    assert tiles2 == tiles
    # tuned and untuned compute the same step (accumulation order only)
    xin = {"x": W.uniform((64, 32, 32, 3), 1, "x")}
    t = W.uniform((64, 10), 2, "t", 4.0, 6.0)
    base = P.CompiledModel(doc, precision=P.PREC_TF32)
    for k in base.weight_shapes:
        base.set_weight(k, m.weight(k))
    l0, g0 = base.gradients(xin, t)
    l1, g1 = m.gradients(xin, t)
    assert abs(l1 - l0) <= 1e-4 * abs(l0)
    for w in g0:
        d = np.linalg.norm(g1[w] - g0[w]) / max(np.linalg.norm(g0[w]), 1e-30)
        assert d < 2e-2, (w, d)
