"""The channel-stationary elementwise path stages its element streams through a
per-thread cp.async ring (ew_codegen.cu, ring_stages): bitwise checks against
float32 numpy restatements (every op is a single IEEE rounding, no FMA) at
sizes whose last grid-stride sweep is partial, for ring depths 3..8, for a
program with too many streams for a ring (register path), and for the
inference-BatchNorm invstd hoist (bitwise the per-element form)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOAD, LOAD_CH, STORE, RELU, ADD, MUL, BN_INFER = 0, 1, 2, 3, 5, 6, 12
EPS = 1e-3


def bn_infer_np(x, m, v, ga, be):
    s = (1.0 / np.sqrt(v.astype(np.float64) + EPS)).astype(np.float32)
    return (((x - m) * s) * ga + be).astype(np.float32)


@pytest.mark.parametrize("rows,C", [(100003, 64), (4099, 512), (33, 4096), (1, 8)])
def test_ring_inference_bn_chain_bitwise(rows, C):
    """Depth-3 chain of inference BatchNorm -> ReLU -> *y -> +y (the C2 mode-A
    shape): 2 element streams in the ring, 12 per-channel operands, the
    variance turned into invstd once per thread."""
    from tests.nncb_ctypes import Dev, ew_run
    rng = np.random.default_rng(rows + C)
    x = rng.uniform(-2, 2, (rows, C)).astype(np.float32)
    y = rng.uniform(-1, 1, (rows, C)).astype(np.float32)
    params = [[rng.uniform(-0.5, 0.5, C).astype(np.float32), rng.uniform(0.2, 2.0, C).astype(np.float32),
               rng.uniform(0.5, 1.5, C).astype(np.float32), rng.uniform(-0.5, 0.5, C).astype(np.float32)]
              for _ in range(3)]
    slots = [Dev(x), Dev(y)] + [Dev(p) for ps in params for p in ps] + [Dev(nbytes=x.nbytes)]
    prog = [dict(op=LOAD, dst=0, slot=0), dict(op=LOAD, dst=1, slot=1)]
    cur, r = 0, 2
    for k in range(3):
        s0 = 2 + 4 * k
        m, v, ga, be = r, r + 1, r + 2, r + 3
        prog += [dict(op=LOAD_CH, dst=m, slot=s0), dict(op=LOAD_CH, dst=v, slot=s0 + 1),
                 dict(op=LOAD_CH, dst=ga, slot=s0 + 2), dict(op=LOAD_CH, dst=be, slot=s0 + 3),
                 dict(op=BN_INFER, dst=r + 4, a=cur, b=m, c=v, d=ga, e=be, imm=EPS),
                 dict(op=RELU, dst=r + 5, a=r + 4), dict(op=MUL, dst=r + 6, a=r + 5, b=1),
                 dict(op=ADD, dst=r + 7, a=r + 6, b=1)]
        cur, r = r + 7, r + 8
    prog.append(dict(op=STORE, a=cur, slot=14))
    ew_run(prog, r, slots, rows * C, C)
    want = x
    for m, v, ga, be in params:
        want = (np.maximum(bn_infer_np(want, m, v, ga, be), 0) * y + y).astype(np.float32)
    got = slots[14].get((rows, C))
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("streams", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("rows,C", [(77777, 128), (515, 64)])
def test_ring_streams_bitwise(streams, rows, C):
    """1..5 element streams (ring depths 8, 6, 4, 3; 5 streams keep the
    register path) with a per-channel scale: out = ((s0 * w) + s1 + ...)."""
    from tests.nncb_ctypes import Dev, ew_run
    rng = np.random.default_rng(streams * 1000 + rows)
    xs = [rng.uniform(-1, 1, (rows, C)).astype(np.float32) for _ in range(streams)]
    w = rng.uniform(0.5, 1.5, C).astype(np.float32)
    slots = [Dev(a) for a in xs] + [Dev(w), Dev(nbytes=xs[0].nbytes)]
    prog = [dict(op=LOAD, dst=i, slot=i) for i in range(streams)]
    prog.append(dict(op=LOAD_CH, dst=streams, slot=streams))
    prog.append(dict(op=MUL, dst=streams + 1, a=0, b=streams))
    acc, r = streams + 1, streams + 2
    for i in range(1, streams):
        prog.append(dict(op=ADD, dst=r, a=acc, b=i))
        acc, r = r, r + 1
    prog.append(dict(op=STORE, a=acc, slot=streams + 1))
    ew_run(prog, r, slots, rows * C, C)
    want = (xs[0] * w).astype(np.float32)
    for a in xs[1:]:
        want = (want + a).astype(np.float32)
    got = slots[streams + 1].get((rows, C))
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
