import sys
sys.path.insert(0, '/root/repo')
import numpy as np
from tests.nncb_ctypes import Dev, GemmDesc, gemm

M, N, K = 128, 64, 32
rng = np.random.default_rng(0)
x = rng.uniform(-1, 1, (M, K)).astype(np.float32)
w = rng.uniform(-1, 1, (K, N)).astype(np.float32)
g = rng.uniform(-1, 1, (M, N)).astype(np.float32)
geo = dict(batch=M, in_f=K, out_f=N)
for kind, a, b, shape, ref in [
    (0, x, w, (M, N), x.astype(np.float64) @ w),          # A K-major, B MN-major
    (1, g, w, (M, K), g.astype(np.float64) @ w.T),        # A K-major, B K-major
    (2, x, g, (K, N), x.T.astype(np.float64) @ g),        # A MN-major, B MN-major
]:
    d = GemmDesc(kind=kind, precision=0, epilogue=0, **geo)
    o = Dev(nbytes=int(np.prod(shape)) * 4)
    gemm(d, Dev(a), Dev(b), None, o)
    tc = o.get(shape)
    err = np.abs(tc - ref).max() / np.abs(ref).max()
    print("kind", kind, "err", err, "tc[0,:3]", tc[0, :3], "ref", ref[0, :3])
    if err > 0.01:
        # is tc a permutation of ref rows/cols?
        rows = [int(np.argmin(np.abs(ref - tc[r]).sum(1))) for r in range(min(8, shape[0]))]
        print("   best-matching ref rows for tc rows 0..7:", rows)
