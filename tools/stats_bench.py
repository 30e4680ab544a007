"""BatchNorm statistics / backward-sum kernels on ResNet-50 shapes (CUDA events)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.nncb_ctypes import K, Dev, ctx, _P

K.nncb_bn_stats.argtypes = [_P, _P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_double]
ev = [ctypes.c_void_p(), ctypes.c_void_p()]
for e in ev:
    K.nncb_event_create(ctypes.byref(e))
for rows, C in [(802816, 64), (802816, 256), (200704, 128), (200704, 512), (50176, 1024), (12544, 2048), (12544, 512)]:
    x = Dev(np.random.default_rng(0).uniform(-1, 1, (rows, C)).astype(np.float32))
    g = Dev(np.random.default_rng(1).uniform(-1, 1, (rows, C)).astype(np.float32))
    st, a, b = Dev(nbytes=2 * C * 4), Dev(nbytes=C * 4), Dev(nbytes=C * 4)
    res = []
    for name, fn, nb in [("stats", lambda: K.nncb_bn_stats(ctx(), x.p, st.p, rows, C, 1e-5), 1),
                         ("grad_reduce", lambda: K.nncb_bn_grad_reduce(ctx(), x.p, st.p, g.p, a.p, b.p, rows, C), 2)]:
        fn()
        K.nncb_event_record(ctx(), ev[0])
        for _ in range(10):
            fn()
        K.nncb_event_record(ctx(), ev[1])
        K.nncb_sync(ctx())
        ms = ctypes.c_float()
        K.nncb_event_elapsed_ms(ev[0], ev[1], ctypes.byref(ms))
        t = ms.value / 10
        res.append(f"{name} {t*1e3:7.1f} us {nb*rows*C*4/t/1e6:6.0f} GB/s")
    print(f"{rows:7d} x {C:5d}: " + " | ".join(res))
