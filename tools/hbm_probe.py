"""HBM ceilings for write-heavy kernels: fill (write only) and copy (read+write), CUDA events."""
import torch
n = 205_520_896   # 822 MB of fp32 (ResNet-50 stage-0 output at batch 256)
x = torch.empty(n, device="cuda")
y = torch.randn(n, device="cuda")
s = torch.randn(n // 4, device="cuda")
for name, fn, nbytes in [("fill", lambda: x.fill_(1.0), 4 * n), ("copy", lambda: x.copy_(y), 8 * n),
                         ("read 1/4 + write", lambda: x.view(4, -1).copy_(s.expand(4, -1)), 4 * n + n)]:
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:18s} {ms*1e3:8.1f} us  {nbytes/ms/1e6:7.0f} GB/s")
