"""The data-parallel exchange path on one GPU: a 1-rank NCCL communicator puts
the real bucketed all-reduce + per-bucket update schedule (runtime::
step_schedule -> nncb_allreduce_sum_on_comm / nncb_sgd_dev on the comm stream,
fork/join events, all captured into the step's CUDA graph) into the training
step. With one rank the all-reduce is the identity, so every loss and every
weight must equal, bit for bit, the same steps of a process without a
communicator. Runs in subprocesses: the communicator is process-wide."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
comm = sys.argv[1] == "1"
if comm:
    P.init_comm(1, 0, P.comm_unique_id())
doc = W.resnet50(8, bn=True, image=64, classes=16)
x = W.uniform((8, 64, 64, 3), 1, "x")
t = W.uniform((8, 16), 2, "t", 0.0, 1.0)
m = P.CompiledModel(doc, precision=P.PREC_TF32)
losses = [m.train_step({"x": x}, t, 0.01)]                       # eager first step
losses += m.train_steps([({"x": x}, t)] * 3, 0.01)               # graph replays, pipelined uploads
losses += m.train_steps([({"x": x}, t)] * 2, 0.005)              # lr change: same graph, device lr
w = {k: m.weight(k) for k in sorted(m.weight_shapes)}
np.savez(sys.argv[2], **w)
with open(sys.argv[2] + ".json", "w") as f:
    json.dump({"losses": losses, "launches": m.launches_per_step()}, f)
"""


def _run(comm, out):
    env = dict(os.environ, NCCL_DEBUG="INFO")
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT, "1" if comm else "0", out],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    with open(out + ".json") as f:
        return json.load(f), r.stdout + r.stderr


def test_one_rank_nccl_step_graph_is_bitwise_the_plain_step(tmp_path):
    import numpy as np
    plain, _ = _run(False, str(tmp_path / "plain"))
    comm, err = _run(True, str(tmp_path / "comm"))
    assert "NCCL INFO" in err   # the communicator really exists
    assert plain["losses"] == comm["losses"]
    # the comm step adds one all-reduce per bucket (NCCL kernels are not nncb launches)
    assert comm["launches"] == plain["launches"]
    a, b = np.load(str(tmp_path / "plain") + ".npz"), np.load(str(tmp_path / "comm") + ".npz")
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
