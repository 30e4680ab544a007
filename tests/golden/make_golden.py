"""Generates tests/golden/* from the REFERENCE implementation (oracle/_ref/libnncref.so,
compiled from /root/reference/proj by oracle/Makefile). Run in the dev container:

    python tests/golden/make_golden.py

Outputs (committed):
  c1_ref.npz          C1 small CNN (no BatchNorm, reference vocabulary), batch 2:
                      input, target, inference output, L1 loss, every weight
                      gradient and the weights after one SGD step (lr 0.05) --
                      all produced by the reference's runtime::execute /
                      train_step on its GEMM_TILED+REF plans.
  known_answers.json  the reference's own hand-computed known answers
                      (tests/test_autodiff.cpp, tests/test_runtime.cpp).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import reference as R  # noqa: E402
from paper_2205_10357_b200 import workloads as W  # noqa: E402


def main():
    doc = W.c1_small_cnn(2, bn=False)
    x = W.uniform((2, 32, 32, 3), 1, "x")
    t = W.uniform((2, 10), 2, "t", 0.0, 1.0)
    m = R.RefModel(doc, 1)
    out = m.run({"x": x})["fc"].astype(np.float32)
    loss, grads = m.gradients({"x": x}, t)
    m2 = R.RefModel(doc, 1)
    step_loss = m2.train_step({"x": x}, t, 0.05)
    arrays = {"x": x, "target": t, "fc": out, "loss": np.array([loss]), "step_loss": np.array([step_loss]),
              "document": np.frombuffer(doc.encode(), dtype=np.uint8)}
    for w, g in grads.items():
        arrays["grad/" + w] = g.astype(np.float32)
    for w in m2.weight_shapes:
        arrays["w0/" + w] = m.weight(w).astype(np.float32)
        arrays["w1/" + w] = m2.weight(w).astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "c1_ref.npz"), **arrays)

    known = {
        "source": "/root/reference/proj/tests (hand-computed known answers)",
        "dense_toy": {"cite": "tests/test_autodiff.cpp:44-73", "W": [[1, 2], [3, 4]], "b": [0, 0], "x": [1, 1],
                      "y": [4, 6], "upstream": [1, 0], "gW": [[1, 0], [1, 0]], "gb": [1, 0], "gx": [1, 3]},
        "relu_backward": {"cite": "tests/test_autodiff.cpp:75-90", "x": [-1, 2], "upstream": [5, 7], "gx": [0, 7]},
        "maxpool_tie": {"cite": "tests/test_autodiff.cpp:199-219", "x": [5, 5], "kernel": [1, 2], "argmax": 0,
                        "upstream": 3, "gx": [3, 0]},
        "l1": {"cite": "tests/test_runtime.cpp:67-75", "p": 2, "t": 0, "loss": 2, "grad": 1},
        "sgd": {"cite": "tests/test_runtime.cpp:100-106", "w": 1, "g": 2, "lr": 0.5, "w_after": 0},
        "fused_chain": {"cite": "tests/test_backends.cpp:246-276", "buffer_intermediates": 0, "fused_registers": 2},
        "alexnet_peak": {"cite": "proj/README.md:121-125", "inference_bytes": 250361792, "training_bytes": 488827200},
    }
    # pin the documented values against the reference run right now
    assert abs(loss - float(np.abs(out.astype(np.float64) - t).mean())) < 1e-6
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(known, f, indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
