"""Synthetic workloads of BASELINE.json as DLB model documents (reference
ingest format, core/src/ingest.cpp:411-500) plus deterministic inputs.

  C1  small CNN: conv(16,3x3,SAME,bias) [BN] ReLU MaxPool2/2, conv(32,...) [BN]
      ReLU MaxPool2/2, Flatten, Dense(10), L1 loss
  C2  depth-16 elementwise chain over two tensors; "bn" mode uses
      4 x [BatchNorm, ReLU, Mul(y), Add(y)], "ref" mode (reference vocabulary)
      4 x [ReLU, Mul(y), Add(y), Add(y)]
  C3/C4 ResNet-50-shaped graph: 7x7/2 stem, 3x3/2 VALID max pool, [3,4,6,3]
      bottlenecks (stride on the 3x3, projection shortcut on the first block),
      residual Add, global average pool, Dense(1000); with or without BatchNorm
  C5  MLP: 8 x [Dense 4096->4096 (bias), GELU, LayerNorm]

Inputs are U(-1,1) from the reference's LCG stream (InitStream, ingest.cpp:43-52)
keyed by (seed, name) when small, or numpy's PCG64 for large tensors (stated).
"""
from __future__ import annotations

import json
from typing import List

import numpy as np

MASK = (1 << 64) - 1


def fnv1a64(text: str) -> int:
    h = 14695981039346656037
    for c in text.encode():
        h ^= c
        h = (h * 1099511628211) & MASK
    return h


def init_stream(seed: int, name: str, n: int, lo: float, hi: float) -> np.ndarray:
    """The reference InitStream (ingest.cpp:43-52), vectorised in numpy uint64."""
    s = np.uint64((seed ^ fnv1a64(name)) & MASK)
    a, c = np.uint64(6364136223846793005), np.uint64(1442695040888963407)
    with np.errstate(over="ignore"):
        s = s * a + c
        # jump-ahead in chunks: state_k = s*a^k + c*(a^k-1)/(a-1); done iteratively per block
        out = np.empty(n, dtype=np.float64)
        block = 4096
        # powers for lanes 1..block
        pa = np.empty(block, dtype=np.uint64)
        pc = np.empty(block, dtype=np.uint64)
        x, y = np.uint64(1), np.uint64(0)
        for k in range(block):
            x = x * a
            y = y * a + c
            pa[k], pc[k] = x, y
        for start in range(0, n, block):
            m = min(block, n - start)
            st = s * pa[:m] + pc[:m]
            out[start:start + m] = (st >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
            s = st[m - 1]
    return lo + out * (hi - lo)


def uniform(shape, seed: int, name: str, lo=-1.0, hi=1.0) -> np.ndarray:
    n = int(np.prod(shape))
    if n <= (1 << 22):
        return init_stream(seed, name, n, lo, hi).astype(np.float32).reshape(shape)
    rng = np.random.Generator(np.random.PCG64(seed ^ (fnv1a64(name) & 0xFFFFFFFF)))
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


def _doc(name, inputs, outputs, nodes, seed=7) -> str:
    return json.dumps({"dialect": "dlb", "name": name, "seed": seed, "inputs": inputs,
                       "outputs": outputs, "nodes": nodes})


def c1_small_cnn(batch: int = 32, bn: bool = True, seed: int = 7) -> str:
    nodes: List[dict] = []

    def block(i, src, filters):
        nodes.append({"name": f"c{i}", "op": "conv2d", "inputs": [src],
                      "attrs": {"filters": filters, "kernel_size": 3, "padding": "same", "use_bias": True}})
        cur = f"c{i}"
        if bn:
            nodes.append({"name": f"bn{i}", "op": "batch_normalization", "inputs": [cur],
                          "attrs": {"epsilon": 1e-3}})
            cur = f"bn{i}"
        nodes.append({"name": f"r{i}", "op": "relu", "inputs": [cur]})
        nodes.append({"name": f"p{i}", "op": "max_pooling2d", "inputs": [f"r{i}"], "attrs": {"pool_size": 2}})
        return f"p{i}"

    x = block(1, "x", 16)
    x = block(2, x, 32)
    nodes.append({"name": "f", "op": "flatten", "inputs": [x]})
    nodes.append({"name": "fc", "op": "dense", "inputs": ["f"], "attrs": {"units": 10}})
    return _doc("c1_small_cnn" + ("_bn" if bn else ""),
                [{"name": "x", "dtype": "f32", "shape": [batch, 32, 32, 3]}], ["fc"], nodes, seed)


def c2_chain(shape=(256, 128, 128, 64), mode: str = "bn", depth: int = 16, seed: int = 7,
             batch_stats: bool = False) -> str:
    """batch_stats: the BatchNorms use batch statistics in every version
    (DLB "training": true) -- the C2 mode-B pass as an inference-role plan,
    without the SaveSet a training forward writes for its backward."""
    pattern = ["bn", "relu", "mul", "add"] if mode == "bn" else ["relu", "mul", "add", "add"]
    nodes, cur = [], "x"
    for k in range(depth):
        op = pattern[k % 4]
        name = f"e{k}_{op}"
        if op == "bn":
            attrs = {"epsilon": 1e-3}
            if batch_stats:
                attrs["training"] = True
            nodes.append({"name": name, "op": "batch_normalization", "inputs": [cur], "attrs": attrs})
        elif op == "relu":
            nodes.append({"name": name, "op": "relu", "inputs": [cur]})
        else:
            nodes.append({"name": name, "op": op, "inputs": [cur, "y"]})
        cur = name
    shp = list(shape)
    return _doc(f"c2_chain_{mode}", [{"name": "x", "dtype": "f32", "shape": shp},
                                     {"name": "y", "dtype": "f32", "shape": shp}], [cur], nodes, seed)


def resnet50(batch: int = 256, bn: bool = True, image: int = 224, classes: int = 1000, seed: int = 7) -> str:
    nodes: List[dict] = []

    def conv(name, src, filters, k, s=1):
        nodes.append({"name": name, "op": "conv2d", "inputs": [src],
                      "attrs": {"filters": filters, "kernel_size": k, "strides": s, "padding": "same",
                                "use_bias": False}})
        cur = name
        if bn:
            nodes.append({"name": name + "_bn", "op": "batch_normalization", "inputs": [cur],
                          "attrs": {"epsilon": 1e-3}})
            cur = name + "_bn"
        return cur

    cur = conv("stem", "x", 64, 7, 2)
    nodes.append({"name": "stem_relu", "op": "relu", "inputs": [cur]})
    nodes.append({"name": "stem_pool", "op": "max_pooling2d", "inputs": ["stem_relu"],
                  "attrs": {"pool_size": 3, "strides": 2}})
    cur = "stem_pool"
    for si, (blocks, width) in enumerate([(3, 64), (4, 128), (6, 256), (3, 512)]):
        for bi in range(blocks):
            p = f"s{si}b{bi}"
            stride = 2 if (bi == 0 and si > 0) else 1
            a = conv(p + "_a", cur, width, 1)
            nodes.append({"name": p + "_a_relu", "op": "relu", "inputs": [a]})
            b = conv(p + "_b", p + "_a_relu", width, 3, stride)
            nodes.append({"name": p + "_b_relu", "op": "relu", "inputs": [b]})
            c = conv(p + "_c", p + "_b_relu", width * 4, 1)
            short = conv(p + "_proj", cur, width * 4, 1, stride) if bi == 0 else cur
            nodes.append({"name": p + "_add", "op": "add", "inputs": [c, short]})
            nodes.append({"name": p + "_out", "op": "relu", "inputs": [p + "_add"]})
            cur = p + "_out"
    nodes.append({"name": "gap", "op": "global_avg_pool2d", "inputs": [cur]})
    nodes.append({"name": "flat", "op": "flatten", "inputs": ["gap"]})
    nodes.append({"name": "fc", "op": "dense", "inputs": ["flat"], "attrs": {"units": classes}})
    return _doc("resnet50" + ("_bn" if bn else ""),
                [{"name": "x", "dtype": "f32", "shape": [batch, image, image, 3]}], ["fc"], nodes, seed)


def mlp(batch: int = 8192, width: int = 4096, layers: int = 8, seed: int = 7) -> str:
    nodes, cur = [], "x"
    for i in range(layers):
        nodes.append({"name": f"d{i}", "op": "dense", "inputs": [cur], "attrs": {"units": width}})
        nodes.append({"name": f"g{i}", "op": "gelu", "inputs": [f"d{i}"]})
        nodes.append({"name": f"ln{i}", "op": "layer_normalization", "inputs": [f"g{i}"],
                      "attrs": {"epsilon": 1e-5}})
        cur = f"ln{i}"
    return _doc("mlp", [{"name": "x", "dtype": "f32", "shape": [batch, width]}], [cur], nodes, seed)
