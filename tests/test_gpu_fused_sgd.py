"""The SGD update fused into the weight-gradient calls at G = 1
(nncb_gemm_desc::sgd_w: the update inside the split-K fold that produces dW,
north star (c) / reference runtime.cpp:485-496): a training step gives
bitwise the weights and losses of the bucket-update schedule
(NNC_NO_FUSED_SGD=1), in every precision mode, through the captured graph and
across learning-rate changes."""
import os
import subprocess
import sys
import json

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, ".")
import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
prec = int(sys.argv[1]); which = sys.argv[2]
if which == "c4":
    doc = W.resnet50(4, bn=True, image=64)
    x = {"x": W.uniform((4, 64, 64, 3), 1, "x")}; t = W.uniform((4, 1000), 2, "t", 4.0, 6.0)
else:
    doc = W.c1_small_cnn(32, bn=True)
    x = {"x": W.uniform((32, 32, 32, 3), 1, "x")}; t = W.uniform((32, 10), 2, "t", 0.0, 1.0)
m = P.CompiledModel(doc, precision=prec)
losses = [m.train_step(x, t, lr) for lr in (1e-3, 1e-3, 5e-4, 1e-3)]
w = {k: m.weight(k).tobytes().hex() for k in sorted(m.weight_shapes)}
print(json.dumps({"losses": losses, "w": w}))
"""


def run(prec, which, fused):
    env = dict(os.environ)
    if not fused:
        env["NNC_NO_FUSED_SGD"] = "1"
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(prec), which], capture_output=True, text=True,
                       env=env, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("which", ["c1", "c4"])
@pytest.mark.parametrize("prec", [0, 1, 2, 3])
def test_fused_sgd_matches_bucket_updates(prec, which):
    if prec == 1 and which == "c4":
        pytest.skip("exact fp32 ResNet step: minutes on the serial-order path")
    a, b = run(prec, which, True), run(prec, which, False)
    assert a["losses"] == b["losses"]
    assert a["w"] == b["w"]
