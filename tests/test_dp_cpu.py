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
