"""Times the LayerNorm backward launches at C5's shape (8192 x 4096) through
the thin C-ABI: dx alone, dgamma, the beta SumRows, and the fused
nncb_layernorm_bwd_params (dx + dgamma + dbeta)."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from tests.nncb_ctypes import K, Dev, ctx  # noqa: E402

P = ctypes.c_void_p
for name, args in [("nncb_layernorm_bwd", [P] * 5 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
                   ("nncb_layernorm_bwd_params", [P] * 7 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
                   ("nncb_layernorm_dgamma", [P] * 4 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
                   ("nncb_sum_rows", [P] * 3 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_int])]:
    getattr(K, name).restype, getattr(K, name).argtypes = ctypes.c_int, args

rows, C = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (8192, 4096)
rng = np.random.default_rng(0)
x, g = Dev(rng.normal(size=(rows, C)).astype(np.float32)), Dev(rng.normal(size=(rows, C)).astype(np.float32))
ga = Dev(rng.uniform(0.5, 1.5, C).astype(np.float32))
gx, dg, db = Dev(nbytes=4 * rows * C), Dev(nbytes=4 * C), Dev(nbytes=4 * C)
c = ctx()


def timeit(fn, reps=50):
    for _ in range(5):
        assert fn() == 0
    e0, e1 = P(), P()
    K.nncb_event_create(ctypes.byref(e0)); K.nncb_event_create(ctypes.byref(e1))
    K.nncb_event_record(c, e0)
    for _ in range(reps):
        fn()
    K.nncb_event_record(c, e1)
    K.nncb_sync(c)
    ms = ctypes.c_float()
    K.nncb_event_elapsed_ms(e0, e1, ctypes.byref(ms))
    return ms.value / reps


mb = rows * C * 4 / 1e6
for label, fn, mbytes in [
        ("ln_bwd dx", lambda: K.nncb_layernorm_bwd(c, x.p, ga.p, g.p, gx.p, rows, C, 1e-5), 3 * mb),
        ("ln_dgamma", lambda: K.nncb_layernorm_dgamma(c, x.p, g.p, dg.p, rows, C, 1e-5), 2 * mb),
        ("sum_rows", lambda: K.nncb_sum_rows(c, g.p, db.p, rows, C, 0), mb),
        ("bwd_params", lambda: K.nncb_layernorm_bwd_params(c, x.p, ga.p, g.p, gx.p, dg.p, db.p, rows, C, 1e-5), 3 * mb)]:
    ms = timeit(fn)
    print(f"{label:12s} {ms * 1e3:8.1f} us  {mbytes / ms / 1e3:7.2f} TB/s")
