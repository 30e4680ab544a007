"""Per-gradient error of the ResNet-50-shaped BN training step vs the float64
oracle (diagnostic; prints one JSON line per precision/batch)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2205_10357_b200 as P
from oracle import restated64 as R64
from paper_2205_10357_b200 import workloads as W


def run(precision, batch, image=224, seed_norm=4, env=None):
    doc = W.resnet50(batch, bn=True, image=image)
    x = W.uniform((batch, image, image, 3), 1, "x")
    t = W.uniform((batch, 1000), 2, "t", 4.0, 6.0)
    m = P.CompiledModel(doc, precision=precision)
    rng = np.random.default_rng(seed_norm)
    for name, shape in m.weight_shapes.items():
        if name.endswith(".gamma"):
            m.set_weight(name, rng.uniform(0.5, 1.5, shape).astype(np.float32))
        elif name.endswith(".beta"):
            m.set_weight(name, rng.uniform(-0.5, 0.5, shape).astype(np.float32))
    weights = {w: m.weight(w) for w in m.weight_shapes}
    o = R64.F64Model(doc, weights)
    oe = R64.F64Model(doc, weights, emulate="tf32" if precision == P.PREC_TF32 else None)
    fwd = m.run({"x": x}, role="train_fwd")
    am = {"stem_pool": fwd["stem_pool.argmax"]}
    # forward value errors along the net
    o.forward({"x": x}, training=True, argmax=am)
    ferr = {}
    for k, v in fwd.items():
        if k in o.values:
            ref = o.values[k]
            ferr[k] = float(np.linalg.norm(v - ref) / max(np.linalg.norm(ref), 1e-30))
    loss, grads = m.gradients({"x": x}, t)
    oloss, og = o.gradients({"x": x}, t, argmax=am)
    gerr = {w: float(np.linalg.norm(grads[w] - g) / max(np.linalg.norm(g), 1e-30)) for w, g in og.items()}
    _, oge = oe.gradients({"x": x}, t, argmax=am)
    eerr = {w: float(np.linalg.norm(grads[w] - g) / max(np.linalg.norm(g), 1e-30)) for w, g in oge.items()
            if np.linalg.norm(g) > 1e-9}
    vg = {}
    return {"precision": precision, "batch": batch, "loss": loss, "oloss": oloss,
            "fwd_worst": sorted(ferr.items(), key=lambda kv: -kv[1])[:8],
            "grad_worst_vs_truth": sorted(gerr.items(), key=lambda kv: -kv[1])[:12],
            "grad_worst_vs_emulated": sorted(eerr.items(), key=lambda kv: -kv[1])[:12],
            "grad_norms": {w: float(np.linalg.norm(g)) for w, g in sorted(og.items(), key=lambda kv: -gerr[kv[0]])[:12]},
            "n_grads": len(og), "n_over_2e-2_vs_emulated": sum(e >= 2e-2 for e in eerr.values())}


if __name__ == "__main__":
    for prec, b in [(P.PREC_TF32, 2), (P.PREC_FP32, 2), (P.PREC_TF32, 8), (P.PREC_TF32, 32)]:
        print(json.dumps(run(prec, b)), flush=True)
