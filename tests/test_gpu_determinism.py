"""Cross-process reproducibility of the tf32 path: the
GEMM tile choice -- which fixes the fp32 accumulation order -- comes from the
committed per-shape table or the static rule, never from timing in the
process, so two processes produce bitwise-identical gradients and losses."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, %r)
import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
assert P._kern.nncb_gemm_tuning_mode() == 1
out = {}
for name, doc, xs, ts in [("c1", W.c1_small_cnn(32, bn=True), (32, 32, 32, 3), (32, 10)),
                          ("rn", W.resnet50(4, bn=True, image=64, classes=16), (4, 64, 64, 3), (4, 16))]:
    m = P.CompiledModel(doc, precision=P.PREC_TF32)
    loss, g = m.gradients({"x": W.uniform(xs, 1, "x")}, W.uniform(ts, 2, "t", 0.0, 1.0))
    out[name + "/loss"] = np.array([loss])
    for k, v in g.items():
        out[name + "/" + k] = v
np.savez(sys.argv[1], **out)
"""


def test_two_processes_give_bitwise_identical_tf32_gradients(tmp_path):
    env = dict(os.environ)
    env.pop("NNCB_TC_AUTOTUNE", None)
    files = []
    for i in range(2):
        f = str(tmp_path / f"run{i}.npz")
        r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT, f], capture_output=True, text=True, timeout=600,
                           env=env)
        assert r.returncode == 0, r.stderr[-3000:]
        files.append(np.load(f))
    a, b = files
    assert sorted(a.files) == sorted(b.files) and len(a.files) > 100
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


FRESH = r"""
import ctypes, sys
sys.path.insert(0, %r)
import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
k = P._kern
assert k.nncb_gemm_tuning_mode() == 3
m = P.CompiledModel(W.c1_small_cnn(32, bn=True), precision=P.PREC_TF32)
m.run({"x": W.uniform((32, 32, 32, 3), 1, "x")})
k.nncb_gemm_tuning_export.restype = ctypes.c_int
k.nncb_gemm_tuning_export.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
n = ctypes.c_size_t()
k.nncb_gemm_tuning_export(None, 0, ctypes.byref(n))
buf = ctypes.create_string_buffer(n.value)
assert k.nncb_gemm_tuning_export(buf, n.value, ctypes.byref(n)) == 0
print(buf.value.decode().count("\n"))
"""


def test_fresh_tuning_measures_shapes_without_the_committed_table():
    """NNCB_TC_AUTOTUNE=fresh (what tools/tune_tiles.py runs): the committed
    table is not consulted, so the C1 inference shapes -- all of which the
    table holds -- are measured in the process and exported."""
    env = dict(os.environ, NNCB_TC_AUTOTUNE="fresh")
    r = subprocess.run([sys.executable, "-c", FRESH % ROOT], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    measured = int(r.stdout.strip().splitlines()[-1])
    assert 0 < measured < 20, measured   # only this process's shapes, not the committed table's 168
