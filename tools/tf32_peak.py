"""Measures the TF32 dense tensor peak with the driver's bf16 recipe (torch
8192^3 matmul, best of 10 and back-to-back for ~4 s), plus this repo's own
tcgen05 GEMM at the same shape in tf32 and bf16 (nncb_gemm, dense forward).
Prints one JSON line; the numbers go to BASELINE.md / profiles/r02."""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def torch_peak(dtype, tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.time()
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            a @ b
        reps += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sustained = 2 * n ** 3 * reps / (e0.elapsed_time(e1) / 1e3) / 1e12
    return best, sustained


def ours(precision):
    from tests.nncb_ctypes import Dev, GemmDesc, K, ctx
    import paper_2205_10357_b200 as P
    n = 8192
    x, w, y = Dev(nbytes=n * n * 4), Dev(nbytes=n * n * 4), Dev(nbytes=n * n * 4)
    d = GemmDesc(kind=0, precision=precision, batch=n, in_f=n, out_f=n)
    assert K.nncb_gemm(ctx(), ctypes.byref(d), x.p, w.p, None, y.p) == 0
    t = P.DeviceTimer()
    t.sync()
    t.start()
    for _ in range(10):
        K.nncb_gemm(ctx(), ctypes.byref(d), x.p, w.p, None, y.p)
    ms = t.stop() / 10
    return 2 * n ** 3 / (ms / 1e3) / 1e12


if __name__ == "__main__":
    tb, ts = torch_peak(torch.float32, True)
    out = {"tf32_tflops_burst": tb, "tf32_tflops_sustained": ts,
           "ours_8192_tf32": ours(0), "ours_8192_bf16_incl_conversion": ours(2),
           "how": "torch.matmul fp32 with allow_tf32, 8192^3, best of 10 (burst) and back to back for 4 s "
                  "(sustained); ours: nncb_gemm dense forward 8192^3, mean of 10"}
    print(json.dumps(out))
