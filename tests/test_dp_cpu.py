"""Data-parallel host arithmetic on CPU with torch.distributed gloo, world size 2
(the only multi-GPU evidence this run can produce: one GPU per gpurun call).

The B200 path shards the batch across ranks, all-reduces (sum) the flat weight-
gradient region and applies SGD with grad_scale = 1/G (runtime.cpp Trainer,
nncb_sgd). For BatchNorm-free graphs a G-rank step must then equal the 1-rank
step on the global batch: the reference L1 loss is a mean over the local batch
(runtime.cpp:474), so mean over ranks of local-mean gradients == global-mean
gradient. This test checks exactly that with the restated oracle's gradients.
"""
import os
import socket

import numpy as np
import pytest

from oracle import restated as O
from paper_2205_10357_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    doc = W.c1_small_cnn(2, bn=False)           # per-rank batch 2 (global 4)
    x = W.uniform((4, 32, 32, 3), 1, "x")[rank * 2:(rank + 1) * 2]
    t = W.uniform((4, 10), 2, "t", 0.0, 1.0)[rank * 2:(rank + 1) * 2]
    m = O.OracleModel(doc)
    _, grads = m.gradients({"x": x}, t)
    names = sorted(grads)
    flat = torch.from_numpy(np.concatenate([grads[k].ravel() for k in names]).astype(np.float64))
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)     # the exchange step (NCCL on the B200 path)
    flat /= world                                   # grad_scale = 1/G in nncb_sgd
    # the unique-id broadcast bench.py uses for ncclCommInitRank
    uid = [b"x" * 128 if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    if rank == 0:
        q.put((names, flat.numpy(), uid[0]))
    dist.destroy_process_group()


@pytest.mark.skipif(not O.available(), reason="oracle/_ref/libnnc_oracle.so not built")
def test_two_rank_gradient_allreduce_equals_global_batch():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    names, flat, uid = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert uid == b"x" * 128
    doc = W.c1_small_cnn(4, bn=False)
    m = O.OracleModel(doc)
    _, g = m.gradients({"x": W.uniform((4, 32, 32, 3), 1, "x")}, W.uniform((4, 10), 2, "t", 0.0, 1.0))
    want = np.concatenate([g[k].ravel() for k in names]).astype(np.float64)
    assert np.max(np.abs(flat - want)) <= 1e-5 * np.max(np.abs(want))


def _check_schedule(s, bucket_elems):
    """Region layout and bucket schedule invariants of runtime::dp_layout."""
    ws = s["weights"]
    off = 0
    for w in ws:   # contiguous, 256-byte aligned, trainable prefix first
        assert w["offset"] == off and w["offset"] % 64 == 0
        off += -(-w["elements"] // 64) * 64
    assert off == s["region_elems"]
    trainable = [w for w in ws if w["grad_launch"] >= 0]
    assert ws[:len(trainable)] == trainable
    assert [w["grad_launch"] for w in trainable] == sorted(w["grad_launch"] for w in trainable)
    end = trainable[-1]["offset"] + trainable[-1]["elements"]
    b = s["buckets"]
    assert b[0]["offset"] == 0 and b[-1]["offset"] + b[-1]["count"] == end
    for x, y in zip(b, b[1:]):
        assert x["offset"] + x["count"] == y["offset"] and x["count"] == bucket_elems
        assert x["close_launch"] <= y["close_launch"]
    for x in b:   # close_launch is the last write of any gradient in the bucket (tight)
        touching = [w["grad_launch"] for w in trainable
                    if w["offset"] < x["offset"] + x["count"] and x["offset"] < w["offset"] + w["elements"]]
        assert x["close_launch"] == max(touching)
        assert 0 <= x["close_launch"] < s["bwd_launches"]


def test_dp_bucket_schedule_resnet():
    """ResNet-50-shaped graph: 32 MB buckets over 25.6M parameters; all but the
    last close before the end of the backward pass, so their all-reduces
    overlap the remaining backward launches."""
    import paper_2205_10357_b200 as P
    s = P.CompiledModel(W.resnet50(2, image=64)).dp_schedule(32 << 20)
    _check_schedule(s, 8 << 20)
    assert len(s["buckets"]) == 4
    assert all(b["close_launch"] < s["bwd_launches"] - 1 for b in s["buckets"][:-1])


def _bucket_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import paper_2205_10357_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    doc = W.c1_small_cnn(2, bn=False)
    x = W.uniform((4, 32, 32, 3), 1, "x")[rank * 2:(rank + 1) * 2]
    t = W.uniform((4, 10), 2, "t", 0.0, 1.0)[rank * 2:(rank + 1) * 2]
    _, grads = O.OracleModel(doc).gradients({"x": x}, t)
    s = P.CompiledModel(doc).dp_schedule(4096)
    region = np.zeros(s["region_elems"], np.float32)
    for w in s["weights"]:
        if w["grad_launch"] >= 0:
            region[w["offset"]:w["offset"] + w["elements"]] = grads[w["name"]].ravel()
    whole = torch.from_numpy(region.copy())
    dist.all_reduce(whole, op=dist.ReduceOp.SUM)
    # the overlapped schedule: each bucket reduced at its close point, in close order
    bucketed = torch.from_numpy(region.copy())
    for b in sorted(s["buckets"], key=lambda b: b["close_launch"]):
        dist.all_reduce(bucketed[b["offset"]:b["offset"] + b["count"]], op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put((s, whole.numpy(), bucketed.numpy()))
    dist.destroy_process_group()


@pytest.mark.skipif(not O.available(), reason="oracle/_ref/libnnc_oracle.so not built")
def test_two_rank_bucketed_allreduce_schedule():
    """gloo, world 2: reducing the gradient region bucket by bucket at the
    dp_layout close points gives the same region as one all-reduce of it."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    s, whole, bucketed = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _check_schedule(s, 1024)
    assert len(s["buckets"]) > 1
    assert np.array_equal(whole, bucketed)
