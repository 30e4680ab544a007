"""Lists the values of a bound C4 training step (debug_keep_values) that no
launch writes -- values whose producer a bind-time fusion pass absorbed. The
launch-by-launch parity harness treats them as unavailable (the oracle's own
value stands in) instead of reading stale arena bytes."""
import sys

sys.path.insert(0, ".")
import paper_2205_10357_b200 as P  # noqa: E402
from paper_2205_10357_b200 import workloads as W  # noqa: E402

doc = W.resnet50(2, bn=True)
x = W.uniform((2, 224, 224, 3), 1, "x")
t = W.uniform((2, 1000), 2, "t", 4.0, 6.0)
m = P.CompiledModel(doc, precision=P.PREC_TF32)
m.debug_keep_values(True)
m.gradients({"x": x}, t)
for role in ("train_fwd", "train_bwd"):
    for v in m.describe[role]["values"]:
        try:
            m.step_value(v["name"])
        except P.NNCError as e:
            if "never written" in str(e):
                print(role, v["name"], v["category"], v["storage"])
