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
    """One rank of a data-parallel training step driven by the Trainer's own
    backward schedule (runtime::step_schedule, the exact action list
    Trainer::enqueue_step issues): walk the backward launches in order, write
    each weight gradient at the launch that produces it (NaN poison at any
    earlier, non-final write), check every weight a launch reads has not been
    updated yet, and run the fork / all-reduce / update actions where the
    schedule puts them (gloo standing in for NCCL)."""
    import torch
    import torch.distributed as dist
    import paper_2205_10357_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    doc = W.c1_small_cnn(2, bn=False)
    x = W.uniform((4, 32, 32, 3), 1, "x")[rank * 2:(rank + 1) * 2]
    t = W.uniform((4, 10), 2, "t", 0.0, 1.0)[rank * 2:(rank + 1) * 2]
    om = O.OracleModel(doc)
    _, grads = om.gradients({"x": x}, t)
    s = P.CompiledModel(doc).step_schedule(4096, comm=True, sgd=True)
    woff = {w["name"]: (w["offset"], w["elements"]) for w in s["weights"]}
    params = np.zeros(s["region_elems"], np.float32)
    for w, (o, n) in woff.items():
        params[o:o + n] = om.w[w].ravel()
    p0 = params.copy()
    gbuf = torch.zeros(s["region_elems"], dtype=torch.float32)
    last_write = {}
    for k, ws in enumerate(s["launch_writes"]):
        for w in ws:
            last_write[w] = k
    lr, scale = 0.05, 1.0 / world
    updated = np.zeros(s["region_elems"], bool)
    stale_reads = []
    acts = {}
    for a in s["actions"]:
        acts.setdefault(a["after"], []).append(a)
    for k in range(s["bwd_launches"]):
        for w in s["launch_reads"][k]:
            o, n = woff[w]
            if updated[o:o + n].any():
                stale_reads.append((k, w))
        for w in s["launch_writes"][k]:
            o, n = woff[w]
            gbuf[o:o + n] = torch.from_numpy(grads[w].ravel()) if last_write[w] == k else float("nan")
        for a in acts.get(k, []):
            if a["kind"] == "allreduce":
                b = s["buckets"][a["bucket"]]
                dist.all_reduce(gbuf[b["offset"]:b["offset"] + b["count"]], op=dist.ReduceOp.SUM)
            elif a["kind"] == "update":
                b = s["buckets"][a["bucket"]]
                sl = slice(b["offset"], b["offset"] + b["count"])
                g = gbuf[sl].numpy().astype(np.float64)
                params[sl] = (params[sl].astype(np.float64) - lr * (g * scale)).astype(np.float32)
                updated[sl] = True
    if rank == 0:
        q.put((s, p0, params, gbuf.numpy().copy(), stale_reads))
    dist.destroy_process_group()


@pytest.mark.skipif(not O.available(), reason="oracle/_ref/libnnc_oracle.so not built")
def test_two_rank_step_schedule_allreduce_and_update():
    """gloo, world 2, the Trainer's backward schedule: every bucket is
    all-reduced only after its last gradient write (no NaN poison survives),
    no backward launch reads a weight after its bucket was updated, and the
    updated region equals SGD of the all-reduced gradients, bit for bit
    (w = (float)((double)w - lr*((double)g_sum * 1/G)), nncb_sgd_dev)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    s, p0, params, gsum, stale = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(s["buckets"]) > 1
    kinds = [a["kind"] for a in s["actions"]]
    assert kinds.count("allreduce") == len(s["buckets"]) == kinds.count("update") and kinds[-1] == "join"
    assert not stale, stale
    assert np.isfinite(gsum).all()
    want = (p0.astype(np.float64) - 0.05 * (gsum.astype(np.float64) * 0.5)).astype(np.float32)
    assert np.array_equal(params, want)
    # the global-batch equivalence of the exchanged gradients
    doc = W.c1_small_cnn(4, bn=False)
    m = O.OracleModel(doc)
    _, g = m.gradients({"x": W.uniform((4, 32, 32, 3), 1, "x")}, W.uniform((4, 10), 2, "t", 0.0, 1.0))
    for w in s["weights"]:
        if w["name"] in g:
            o, n = w["offset"], w["elements"]
            ref = g[w["name"]].ravel().astype(np.float64)
            assert np.max(np.abs(gsum[o:o + n] * 0.5 - ref)) <= 1e-5 * max(np.max(np.abs(ref)), 1e-12), w["name"]


def test_step_schedule_update_points_resnet():
    """runtime::step_schedule on the ResNet-50-shaped graph: every bucket is
    all-reduced at its close point and updated no earlier than the last
    backward launch that reads any of its weights; without a communicator the
    same updates fork off the compute stream; without the update nothing but
    the all-reduces remains; the compute stream always joins last."""
    import paper_2205_10357_b200 as P
    m = P.CompiledModel(W.resnet50(2, image=64))
    s = m.step_schedule(32 << 20, comm=True, sgd=True)
    woff = {w["name"]: (w["offset"], w["elements"]) for w in s["weights"]}
    last_read = {}
    for k, ws in enumerate(s["launch_reads"]):
        for w in ws:
            last_read[w] = k
    for i, b in enumerate(s["buckets"]):
        touching = [w for w, (o, n) in woff.items() if o < b["offset"] + b["count"] and b["offset"] < o + n]
        assert b["update_launch"] >= b["close_launch"]
        assert all(b["update_launch"] >= last_read.get(w, -1) for w in touching)
        acts = [a for a in s["actions"] if a["bucket"] == i]
        assert [a["kind"] for a in acts] == ["allreduce", "update"]
        assert acts[0]["after"] == b["close_launch"] and acts[1]["after"] == b["update_launch"]
    assert s["actions"][-1]["kind"] == "join"
    local = m.step_schedule(32 << 20, comm=False, sgd=True)
    assert [a["kind"] for a in local["actions"] if a["kind"] in ("allreduce", "update")] == \
        ["update"] * len(s["buckets"])
    nosgd = m.step_schedule(32 << 20, comm=True, sgd=False)
    assert [a["kind"] for a in nosgd["actions"] if a["kind"] in ("allreduce", "update")] == \
        ["allreduce"] * len(s["buckets"])
    assert m.step_schedule(32 << 20, comm=False, sgd=False)["actions"] == []
