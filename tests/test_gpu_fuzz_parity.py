"""Random graphs through every bind-time fusion pass, launch by launch.

The runtime rewrites the bound step (BatchNorm statistics into GEMM
epilogues, BN backward reductions and bias gradients into the groups that
store their gradient, LayerNorm parameter gradients into its backward, the
inference BN affine into GEMM epilogues) by matching producers and checking
hazards on ARENA BYTES, which the planner reuses between values with disjoint
lifetimes. Fixed topologies exercise only the reuse patterns they happen to
produce; these graphs draw random mixes of conv (1x1 / 3x3, stride 1 / 2) +
BatchNorm + ReLU / GELU chains, residual joins (BN after the join or on the
branch), pre-activation blocks, pooling and a Dense + LayerNorm head, and
check the training step launch by launch (oracle.restated64.local_parity)
against the precision-emulating float64 oracle, plus the inference plan
(BN affine in the GEMM epilogue) against the oracle in inference mode."""
import json

import numpy as np
import pytest

import paper_2205_10357_b200 as P
from oracle import restated64 as R64
from paper_2205_10357_b200 import workloads as W
from tests.test_gpu_baseline_parity import device_reader, randomize_norms

pytestmark = pytest.mark.gpu


def random_graph(seed, batch=4, hw=16, c0=32):
    rng = np.random.default_rng(seed)
    nodes, k = [], [0]

    def add(op, ins, **attrs):
        k[0] += 1
        name = f"n{k[0]}_{op[:4]}"
        d = {"name": name, "op": op, "inputs": ins}
        if attrs:
            d["attrs"] = attrs
        nodes.append(d)
        return name

    def conv(src, filters, ksz, s=1, bias=False):
        return add("conv2d", [src], filters=filters, kernel_size=ksz, strides=s, padding="same", use_bias=bias)

    def bn(src):
        return add("batch_normalization", [src], epsilon=1e-3)

    cur, c, h = "x", c0, hw
    cur = bn(conv(cur, c, 3, 1, bool(rng.integers(2))))
    cur = add("relu", [cur])
    for _ in range(int(rng.integers(3, 6))):
        kind = int(rng.integers(5))
        if kind == 0:      # plain conv-BN-act
            cur = bn(conv(cur, c, int(rng.choice([1, 3]))))
            cur = add("relu" if rng.integers(2) else "gelu", [cur])
        elif kind == 1:    # bottleneck with a residual join, BN before the join
            s = 2 if (h >= 8 and rng.integers(2)) else 1
            co = int(rng.choice([c, 2 * c]))
            a = add("relu", [bn(conv(cur, c, 1))])
            b = add("relu", [bn(conv(a, c, 3, s))])
            m = bn(conv(b, co, 1))
            short = bn(conv(cur, co, 1, s)) if (s != 1 or co != c) else cur
            cur = add("relu", [add("add", [m, short])])
            c, h = co, (h + s - 1) // s
        elif kind == 2:    # pre-activation: BN fed by an elementwise join
            a = conv(add("relu", [bn(cur)]), c, 3)
            cur = add("add", [a, cur])
        elif kind == 3:    # gating: mul of two branches
            a = bn(conv(cur, c, 1))
            b = add("relu", [bn(conv(cur, c, 3))])
            cur = add("relu", [add("mul", [a, b])])
        else:              # downsample by pooling
            if h >= 8:
                cur = add("max_pooling2d", [cur], pool_size=2, strides=2)
                h //= 2
            cur = add("relu", [bn(conv(cur, c, 1, 1, True))])
    cur = add("global_avg_pool2d", [cur])
    cur = add("flatten", [cur])
    cur = add("dense", [cur], units=64)
    cur = add("layer_normalization", [cur], epsilon=1e-5)
    cur = add("gelu", [cur])
    cur = add("dense", [cur], units=10)
    return json.dumps({"dialect": "dlb", "name": f"fuzz{seed}", "seed": 7,
                       "inputs": [{"name": "x", "dtype": "f32", "shape": [batch, hw, hw, c0]}],
                       "outputs": [cur], "nodes": nodes})


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("precision,emulate,tol", [(P.PREC_TF32, "tf32", 2e-3), (P.PREC_BF16, "bf16", 2e-3),
                                                    (P.PREC_TF32X3, None, 1e-4)])
def test_random_graph_step_launch_by_launch(seed, precision, emulate, tol):
    doc = random_graph(seed)
    x = W.uniform((4, 16, 16, 32), 1 + seed, "x")
    t = W.uniform((4, 10), 2 + seed, "t", 4.0, 6.0)
    m = P.CompiledModel(doc, precision=precision)
    randomize_norms(m, np.random.default_rng(seed))
    m.debug_keep_values(True)
    _, grads = m.gradients({"x": x}, t)
    weights = {w: m.weight(w) for w in m.weight_shapes}
    res = R64.local_parity(R64.F64Model(doc, weights, emulate=emulate), {"x": x}, device_reader(m), grads, t)
    assert len(res["weights"]) == len(grads)
    bad = {part: {k: e for k, e in res[part].items() if not e < tol} for part in res}
    assert not any(bad.values()), bad
    m.debug_keep_values(False)


@pytest.mark.parametrize("seed", range(8))
def test_random_graph_inference_launch_by_launch(seed):
    doc = random_graph(seed)
    x = W.uniform((4, 16, 16, 32), 1 + seed, "x")
    m = P.CompiledModel(doc, precision=P.PREC_TF32)
    rng = np.random.default_rng(seed)
    randomize_norms(m, rng)
    for name, shape in m.weight_shapes.items():   # moving statistics away from (0, 1)
        if name.endswith(".moving_mean"):
            m.set_weight(name, rng.uniform(-0.2, 0.2, shape).astype(np.float32))
        elif name.endswith(".moving_variance"):
            m.set_weight(name, rng.uniform(0.5, 2.0, shape).astype(np.float32))
    m.debug_keep_values(True)
    m.run({"x": x})

    def value(name):
        try:
            return m.run_value(name)
        except P.NNCError:
            return None

    weights = {w: m.weight(w) for w in m.weight_shapes}
    res = R64.local_forward_parity(R64.F64Model(doc, weights, emulate="tf32"), {"x": x}, value)
    assert len(res) >= 5
    bad = {k: e for k, e in res.items() if not e < 2e-3}
    assert not bad, bad
    m.debug_keep_values(False)
