"""HBM bandwidth by traffic mix, with torch kernels only (not this repo's): the
driver's copy figure (MEASURED_PEAKS.json: b.copy_(a), read + write bytes) is
the right denominator for a read-write stream, but a read-dominated pass (the
C2 statistics pass reads two tensors and writes nothing) can exceed it. This
measures, best of 10 with CUDA events over 1 Gi fp32 elements:
  copy:      b.copy_(a)              (read + write bytes, the driver's recipe)
  read:      torch.sum(a)            (read bytes)
  read2:     torch.dot(a, b)         (two read streams)
  read2w1:   torch.add(a, b, out=c)  (two reads, one write)
  read2w1_c4_stage1: the same at 200704 x 128 elements (one C4 stage-1 tensor)
Prints one JSON line (profiles/r02/hbm_mix_peaks.json)."""
import json

import torch


def best_gbs(fn, nbytes, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def main():
    n = 1 << 30
    a = torch.rand(n, device="cuda")
    b = torch.rand(n, device="cuda")
    c = torch.empty(n, device="cuda")
    e = 4 * n
    out = {
        "copy_gbs": best_gbs(lambda: b.copy_(a), 2 * e),
        "read_gbs": best_gbs(lambda: torch.sum(a), e),
        "read2_gbs": best_gbs(lambda: torch.dot(a, b), 2 * e),
        "read2w1_gbs": best_gbs(lambda: torch.add(a, b, out=c), 3 * e),
        "how": "torch kernels, 1 Gi fp32 elements per tensor, best of 10, CUDA events; bytes = tensors read + written",
        "gpu": torch.cuda.get_device_name(0),
    }
    # the same 2-read / 1-write kernel at the C4 stage-1 activation size
    # (200704 x 128 = 25.7 M elements): launch ramp and tail cost a visible
    # share of a ~50 us kernel, so the fused groups' rate at that size is
    # compared against this, not against the 1 Gi figure
    m = 200704 * 128
    a2, b2, c2 = a[:m], b[:m], c[:m]
    out["read2w1_c4_stage1_gbs"] = best_gbs(lambda: torch.add(a2, b2, out=c2), 3 * 4 * m, reps=20)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
