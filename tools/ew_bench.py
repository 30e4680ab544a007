"""Fused elementwise kernel timing: relu-grad group with / without the fused
BatchNorm backward reduction (REDUCE_BN_GRAD), CUDA events, one shape."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.nncb_ctypes import K, Dev, EwInstr, EwProgram, ctx, _P

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=200704)
ap.add_argument("--C", type=int, default=128)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--prog", default="relu_grad", choices=["relu_grad", "bngrad", "bngrad_fast"])
args = ap.parse_args()
rows, C = args.rows, args.C
rng = np.random.default_rng(0)
g = Dev(rng.uniform(-1, 1, (rows, C)).astype(np.float32))
m = Dev(rng.uniform(-1, 1, (rows, C)).astype(np.float32))
x = Dev(rng.uniform(-1, 1, (rows, C)).astype(np.float32))
mean, inv = Dev(np.zeros(C, np.float32)), Dev(np.ones(C, np.float32))
out = Dev(nbytes=rows * C * 4)
sg, sgx = Dev(rng.uniform(-1, 1, C).astype(np.float32)), Dev(rng.uniform(-1, 1, C).astype(np.float32))
LOAD, LOAD_CH, STORE, RG, RED = 0, 1, 2, 4, 13
base = [dict(op=LOAD, dst=0, slot=0), dict(op=LOAD, dst=1, slot=1), dict(op=RG, dst=2, a=1, b=0),
        dict(op=STORE, a=2, slot=2)]
red = [dict(op=LOAD, dst=3, slot=3), dict(op=LOAD_CH, dst=4, slot=4), dict(op=LOAD_CH, dst=5, slot=5),
       dict(op=RED, a=2, b=3, c=4, d=5, slot=6, e=7)]
ev = [ctypes.c_void_p(), ctypes.c_void_p()]
for e in ev:
    K.nncb_event_create(ctypes.byref(e))
gamma = Dev(np.ones(C, np.float32))
BNG = 14 if args.prog == "bngrad_fast" else 11
bng = [dict(op=LOAD, dst=0, slot=0), dict(op=LOAD, dst=1, slot=1), dict(op=LOAD_CH, dst=2, slot=2),
       dict(op=LOAD_CH, dst=3, slot=3), dict(op=LOAD_CH, dst=4, slot=4), dict(op=LOAD_CH, dst=5, slot=5),
       dict(op=LOAD_CH, dst=6, slot=6), dict(op=BNG, dst=7, a=0, b=1, c=2, d=3, e=4, f=5, h=6, imm=float(rows)),
       dict(op=STORE, a=7, slot=7)]
cases = ([("relu_grad", base, [g, m, out], 3), ("relu_grad+reduce", base + red, [g, m, out, x, mean, inv, sg, sgx], 4)]
         if args.prog == "relu_grad" else [("bn_grad", bng, [x, g, mean, inv, gamma, sg, sgx, out], 3)])
for name, prog, slots, nbytes in cases:
    arr = (EwInstr * len(prog))(*[EwInstr(**i) for i in prog])
    p = EwProgram(len(prog), arr, 8, len(slots))
    kern = _P()
    assert K.nncb_ew_compile(ctx(), ctypes.byref(p), ctypes.byref(kern)) == 0
    ptrs = (_P * len(slots))(*[s.p for s in slots])
    K.nncb_ew_launch(ctx(), kern, ptrs, rows * C, C)
    K.nncb_event_record(ctx(), ev[0])
    for _ in range(args.reps):
        K.nncb_ew_launch(ctx(), kern, ptrs, rows * C, C)
    K.nncb_event_record(ctx(), ev[1])
    K.nncb_sync(ctx())
    ms = ctypes.c_float()
    K.nncb_event_elapsed_ms(ev[0], ev[1], ctypes.byref(ms))
    t = ms.value / args.reps
    print(f"{name:18s} {t*1e3:8.1f} us  {nbytes*rows*C*4/t/1e6:7.0f} GB/s")
