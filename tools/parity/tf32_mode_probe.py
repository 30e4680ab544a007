"""Which fp32 -> tf32 operand conversion do the tcgen05 kind::tf32 GEMMs
perform? Compare one dense layer (and one conv) of the product path against
numpy with truncated vs round-to-nearest tf32 operands (diagnostic)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2205_10357_b200 as P
from oracle import restated64 as R64
from paper_2205_10357_b200 import workloads as W


def tf32(a, mode):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    if mode == "rn":
        u = u + np.uint32(0x1000)
    return (u & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)


doc = json.dumps({"dialect": "dlb", "name": "d", "seed": 1,
                  "inputs": [{"name": "x", "dtype": "f32", "shape": [512, 1024]}], "outputs": ["y"],
                  "nodes": [{"name": "y", "op": "dense", "inputs": ["x"], "attrs": {"units": 256, "use_bias": False}}]})
x = W.uniform((512, 1024), 1, "x")
m = P.CompiledModel(doc, precision=P.PREC_TF32)
w = m.weight("y.weight")
y = m.run({"x": x})["y"].astype(np.float64)
for mode in ("trunc", "rn"):
    ref = tf32(x, mode) @ tf32(w, mode)
    print("dense", mode, float(np.max(np.abs(y - ref)) / np.max(np.abs(ref))))
print("dense exact-f64", float(np.max(np.abs(y - x.astype(np.float64) @ w)) / np.max(np.abs(y))))
doc = W.resnet50(2, bn=False, image=32, classes=16)
d = json.loads(doc)
d["nodes"] = d["nodes"][:1]
d["outputs"] = ["stem"]
doc = json.dumps(d)
x = W.uniform((2, 32, 32, 3), 1, "x")
m = P.CompiledModel(doc, precision=P.PREC_TF32)
wt = m.weight("stem.weight")
y = m.run({"x": x})["stem"].astype(np.float64)
for mode in ("trunc", "rn"):
    ref = R64.conv2d(tf32(x, mode), tf32(wt, mode), None, (2, 2), True)
    print("stem", mode, float(np.max(np.abs(y - ref)) / np.max(np.abs(ref))))
