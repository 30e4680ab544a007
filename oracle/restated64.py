"""oracle/restated64.py -- TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the hot path, used as the "truth" against which
the B200 tf32 path (and the float32 oracles) are measured on BASELINE-shaped
graphs that the per-element C restatement is too slow for (ResNet-50-shaped at
224x224, C5 at 8192x4096).

It walks the same DLB documents as oracle/restated.py and restates the
reference formulas in float64 with vectorised numpy:
  conv2d (+grad input/weight, TF-SAME/VALID)  kernels.hpp:166-243, geometry kernels.cpp:12-53
  dense (+grads), sum_cols / sum_nhw          kernels.hpp:118-160, 245-250
  maxpool2d (+grad; argmax = first max in window scan order)  kernels.hpp:258-302
  adaptive_avg_pool2d (+grad)                 kernels.hpp:304-344
  relu / relu_grad / add / mul                kernels.hpp:47-70
  l1_loss, sgd                                runtime.cpp:468-496
  autodiff fan-out accumulation (Add)         autodiff.cpp:69-78
Extension ops (the reference has none; formulas as in oracle/nnc_oracle.c):
  BatchNorm (training statistics, biased variance; inference moving stats),
  GELU (erf form), LayerNorm, softmax cross-entropy.

Pinning (tests/test_oracle.py):
  * reference-vocabulary graphs: against the reference itself run in float64
    (oracle/_ref/libnncref.so, whose runtime is dtype-generic, runtime.cpp:425-434);
  * extension ops: against torch.nn.functional in float64 (an independent
    implementation) and against central finite differences (autodiff.cpp:325-400).

Options a parity test may use:
  emulate = "bf16": the device's bf16 mode -- the forward / input-gradient
           operands of contractions on the bf16 route (bf16_route: aligned
           K blocks, arithmetic intensity >= 128) rounded to nearest at bf16,
           every other tensor-core operand truncated to tf32, fp32 storage;
  emulate = "tf32" (constructor): the arithmetic of the device's tf32 mode,
           restated -- every stored value rounded to float32, and every GEMM
           operand truncated to tf32 (1+8+10 bits: tcgen05 kind::tf32 reads the
           fp32 pattern's top 19 bits; measured by tools/parity/tf32_mode_probe.py)
           for layers with >= 16 output channels (narrower ones run the exact
           fp32 path on the device). Products and sums stay float64, so what
           remains against the device is accumulation order. The default
           (None) is the float64 truth.
  argmax = {pool_name: float window-linear index array} replaces the pool's own
           argmax (feed the device's indices so near-ties cannot move entries);
  loss   = "l1" (reference) or "softmax_ce" (extension, target = probabilities).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import json
import math
from typing import Dict, Optional

import numpy as np

MASK = (1 << 64) - 1


def _pair(a, key, default=None):
    v = a.get(key, default)
    return (v, v) if isinstance(v, int) else tuple(v)


# --------------------------------------------------------------------------
# deterministic initializer: InitStream (reference ingest.cpp:43-70), the LCG
# stepped with a closed-form jump-ahead so large weights initialise fast
# --------------------------------------------------------------------------

def fnv1a64(text: str) -> int:
    h = 14695981039346656037
    for c in text.encode():
        h = ((h ^ c) * 1099511628211) & MASK
    return h


_A, _C = 6364136223846793005, 1442695040888963407


def init_uniform(seed: int, name: str, n: int, lo: float, hi: float) -> np.ndarray:
    s = (seed ^ fnv1a64(name)) & MASK
    s = (s * _A + _C) & MASK
    out = np.empty(n, dtype=np.float64)
    block = 4096
    pa = np.empty(block, dtype=np.uint64)
    pc = np.empty(block, dtype=np.uint64)
    x, y = 1, 0
    for k in range(block):   # state after k+1 steps: s*A^(k+1) + C*(A^k + ... + 1)
        x = (x * _A) & MASK
        y = (y * _A + _C) & MASK
        pa[k], pc[k] = x, y
    st = np.uint64(s)
    with np.errstate(over="ignore"):
        for start in range(0, n, block):
            m = min(block, n - start)
            v = st * pa[:m] + pc[:m]
            out[start:start + m] = (v >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
            st = v[m - 1]
    return lo + out * (hi - lo)


def init_weight(seed, name, shape, fan_in):
    b = 1.0 / math.sqrt(fan_in)
    return init_uniform(seed, name, int(np.prod(shape)), -b, b).astype(np.float32).reshape(shape)


# --------------------------------------------------------------------------
# geometry (kernels.cpp:12-53)
# --------------------------------------------------------------------------

def tf32_trunc(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32).astype(np.float64)


def f32_round(a):
    return np.asarray(a, np.float32).astype(np.float64)


def bf16_round(a):
    """Round to nearest even at bf16 (what the device's fp32 -> bf16 operand
    conversion does, __float2bfloat16_rn)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def bf16_route(K, Ck, N, kind, taps):
    """The device's NNCB_PREC_BF16 route rule (gemm_tc.cu bf16_eligible): forward
    and input-gradient contractions with aligned K blocks whose arithmetic
    intensity K*N / (2*(Ck + N)) reaches 128; dense weight gradients
    ("dense_wgrad": K = batch, Ck = in, N = out) when in*out / (2*(in + out))
    reaches 128 (they run over transposed copies); convolution weight
    gradients never."""
    if kind == "wgrad":
        return False
    if kind == "dense_wgrad":
        return K % 8 == 0 and Ck % 8 == 0 and N % 8 == 0 and Ck * N / (2.0 * (Ck + N)) >= 128.0
    aligned = Ck % 8 == 0 and N % 8 == 0 if taps == 1 else Ck % 64 == 0
    return aligned and K * N / (2.0 * (Ck + N)) >= 128.0


def conv_geom(xd, k, s, same):
    n, ih, iw, ci = xd
    if same:
        oh, ow = -(-ih // s[0]), -(-iw // s[1])
        ph = max((oh - 1) * s[0] + k[0] - ih, 0)
        pw = max((ow - 1) * s[1] + k[1] - iw, 0)
        return oh, ow, (ph // 2, ph - ph // 2), (pw // 2, pw - pw // 2)
    return (ih - k[0]) // s[0] + 1, (iw - k[1]) // s[1] + 1, (0, 0), (0, 0)


def _windows(xp, kh, kw, sh, sw, oh, ow):
    """[n, oh, ow, kh, kw, c] strided view of a (padded) NHWC tensor."""
    n, H, W, c = xp.shape
    st = xp.strides
    return np.lib.stride_tricks.as_strided(
        xp, shape=(n, oh, ow, kh, kw, c),
        strides=(st[0], st[1] * sh, st[2] * sw, st[1], st[2], st[3]), writeable=False)


def conv2d(x, w, b, s, same):
    kh, kw, ci, co = w.shape
    oh, ow, ph, pw = conv_geom(x.shape, (kh, kw), s, same)
    xp = np.pad(x, ((0, 0), ph, pw, (0, 0)))
    cols = np.ascontiguousarray(_windows(xp, kh, kw, s[0], s[1], oh, ow)).reshape(-1, kh * kw * ci)
    y = (cols @ w.reshape(-1, co)).reshape(x.shape[0], oh, ow, co)
    return y + b if b is not None else y


def conv2d_grad_input(gy, w, xshape, s, same):
    kh, kw, ci, co = w.shape
    n, ih, iw, _ = xshape
    oh, ow, ph, pw = conv_geom(xshape, (kh, kw), s, same)
    gp = np.zeros((n, ih + ph[0] + ph[1] + s[0], iw + pw[0] + pw[1] + s[1], ci))
    g2 = gy.reshape(-1, co)
    for dh in range(kh):
        for dw in range(kw):
            gp[:, dh:dh + s[0] * oh:s[0], dw:dw + s[1] * ow:s[1], :] += (g2 @ w[dh, dw].T).reshape(n, oh, ow, ci)
    return gp[:, ph[0]:ph[0] + ih, pw[0]:pw[0] + iw, :]


def conv2d_grad_weight(x, gy, kshape, s, same):
    kh, kw, ci, co = kshape
    oh, ow, ph, pw = conv_geom(x.shape, (kh, kw), s, same)
    xp = np.pad(x, ((0, 0), ph, pw, (0, 0)))
    g2 = gy.reshape(-1, co)
    gw = np.empty(kshape)
    for dh in range(kh):
        for dw in range(kw):
            xs = xp[:, dh:dh + s[0] * oh:s[0], dw:dw + s[1] * ow:s[1], :][:, :oh, :ow, :]
            gw[dh, dw] = xs.reshape(-1, ci).T @ g2
    return gw


def maxpool2d(x, k, s):
    n, ih, iw, c = x.shape
    oh, ow = (ih - k[0]) // s[0] + 1, (iw - k[1]) // s[1] + 1
    win = _windows(x, k[0], k[1], s[0], s[1], oh, ow)           # [n,oh,ow,kh,kw,c]
    flat = np.moveaxis(win, 5, 3).reshape(n, oh, ow, c, k[0] * k[1])
    idx = np.argmax(flat, axis=-1)                               # first max in scan order
    y = np.take_along_axis(flat, idx[..., None], axis=-1)[..., 0]
    return y, idx.astype(np.float64)


def maxpool_gather(x, idx, k, s):
    """Pool output for given window-linear indices (device-fed argmax)."""
    n, ih, iw, c = x.shape
    oh, ow = idx.shape[1], idx.shape[2]
    win = _windows(x, k[0], k[1], s[0], s[1], oh, ow)
    flat = np.moveaxis(win, 5, 3).reshape(n, oh, ow, c, k[0] * k[1])
    return np.take_along_axis(flat, idx.astype(np.int64)[..., None], axis=-1)[..., 0]


def maxpool2d_grad(idx, gy, xshape, k, s):
    n, ih, iw, c = xshape
    oh, ow = gy.shape[1], gy.shape[2]
    gx = np.zeros(xshape)
    wi = idx.astype(np.int64)
    for dh in range(k[0]):
        for dw in range(k[1]):
            sel = np.where(wi == dh * k[1] + dw, gy, 0.0)
            gx[:, dh:dh + s[0] * oh:s[0], dw:dw + s[1] * ow:s[1], :][:, :oh, :ow, :] += sel
    return gx


def _abounds(o, i, out):
    return (o * i) // out, ((o + 1) * i + out - 1) // out


def avgpool(x, oh, ow):
    n, ih, iw, c = x.shape
    y = np.empty((n, oh, ow, c))
    for o in range(oh):
        h0, h1 = _abounds(o, ih, oh)
        for p in range(ow):
            w0, w1 = _abounds(p, iw, ow)
            y[:, o, p, :] = x[:, h0:h1, w0:w1, :].sum(axis=(1, 2)) / ((h1 - h0) * (w1 - w0))
    return y


def avgpool_grad(gy, xshape):
    n, ih, iw, c = xshape
    oh, ow = gy.shape[1], gy.shape[2]
    gx = np.zeros(xshape)
    for o in range(oh):
        h0, h1 = _abounds(o, ih, oh)
        for p in range(ow):
            w0, w1 = _abounds(p, iw, ow)
            gx[:, h0:h1, w0:w1, :] += (gy[:, o, p, :] / ((h1 - h0) * (w1 - w0)))[:, None, None, :]
    return gx


def bn_stats(x2, eps):
    mean = x2.mean(axis=0)
    var = np.maximum((x2 * x2).mean(axis=0) - mean * mean, 0.0)
    return mean, 1.0 / np.sqrt(var + eps)


def gelu(x):
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def gelu_grad(x, g):
    from scipy.special import erf
    cdf = 0.5 * (1.0 + erf(x / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return g * (cdf + x * pdf)


def l1_loss(p, t):
    d = p - t
    n = p.size
    return float(np.abs(d).sum() / n), np.sign(d) / n


def softmax_ce(logits, t):
    """loss = -sum_r sum_c t[r,c] log softmax(z)[r,c] / rows; grad = (softmax(z) - t)/rows
    (target rows are probability vectors)."""
    z = logits.reshape(-1, logits.shape[-1])
    tt = t.reshape(z.shape)
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    ssum = e.sum(axis=1, keepdims=True)
    logp = (z - m) - np.log(ssum)
    rows = z.shape[0]
    loss = float(-(tt * logp).sum() / rows)
    grad = (e / ssum - tt) / rows
    return loss, grad.reshape(logits.shape)


class F64Model:
    """A DLB document evaluated in float64 (weights are given as float32 or
    float64 arrays and promoted; missing ones are initialised like ingest)."""

    def __init__(self, document: str, weights: Optional[Dict[str, np.ndarray]] = None,
                 emulate: Optional[str] = None):
        if emulate not in (None, "tf32", "bf16"):
            raise ValueError(emulate)
        self.emulate = emulate
        d = json.loads(document)
        self.seed = d.get("seed", 0)
        self.nodes = d["nodes"]
        self.outputs = d["outputs"]
        self.inputs = {i["name"]: tuple(i["shape"]) for i in d["inputs"]}
        weights = weights or {}
        self.w: Dict[str, np.ndarray] = {}
        dims = dict(self.inputs)

        def wt(name, shape, fan_in):
            if name in weights:
                self.w[name] = np.asarray(weights[name], dtype=np.float64).reshape(shape)
            else:
                self.w[name] = init_weight(self.seed, name, shape, fan_in).astype(np.float64)

        for n in self.nodes:
            op, name, a = n["op"], n["name"], n.get("attrs", {})
            x = dims[n["inputs"][0]] if n.get("inputs") else None
            if op == "conv2d":
                k, s = _pair(a, "kernel_size"), _pair(a, "strides", 1)
                co = a["filters"]
                wt(name + ".weight", (k[0], k[1], x[3], co), k[0] * k[1] * x[3])
                if a.get("use_bias", True):
                    wt(name + ".bias", (co,), k[0] * k[1] * x[3])
                oh, ow, _, _ = conv_geom(x, k, s, a.get("padding", "valid") == "same")
                dims[name] = (x[0], oh, ow, co)
            elif op == "dense":
                u = a["units"]
                wt(name + ".weight", (x[1], u), x[1])
                if a.get("use_bias", True):
                    wt(name + ".bias", (u,), x[1])
                dims[name] = (x[0], u)
            elif op == "max_pooling2d":
                k = _pair(a, "pool_size")
                s = _pair(a, "strides") if "strides" in a else k
                dims[name] = (x[0], (x[1] - k[0]) // s[0] + 1, (x[2] - k[1]) // s[1] + 1, x[3])
            elif op == "global_avg_pool2d":
                dims[name] = (x[0], 1, 1, x[3])
            elif op == "flatten":
                dims[name] = (x[0], int(np.prod(x[1:])))
            elif op in ("batch_normalization", "layer_normalization"):
                c = x[-1]
                for suffix, init in ((".gamma", 1.0), (".beta", 0.0)):
                    self.w[name + suffix] = np.asarray(weights.get(name + suffix, np.full(c, init)), np.float64)
                if op == "batch_normalization":
                    self.w[name + ".moving_mean"] = np.asarray(weights.get(name + ".moving_mean", np.zeros(c)),
                                                               np.float64)
                    self.w[name + ".moving_variance"] = np.asarray(
                        weights.get(name + ".moving_variance", np.ones(c)), np.float64)
                dims[name] = x
            else:
                dims[name] = x
        self.dims = dims

    def _st(self, a):
        """A stored value: float32-rounded under emulation."""
        return f32_round(a) if self.emulate else a

    def _op(self, a, co, route=None):
        """A GEMM operand of a layer with `co` output channels; route = (K, Ck,
        N, kind, taps) of the contraction, for the bf16 mode's route rule."""
        if not self.emulate or co < 16:
            return a
        if self.emulate == "bf16" and route is not None and bf16_route(*route):
            return bf16_round(a)
        return tf32_trunc(a)

    # ------------------------------------------------------------ per node
    def node_forward(self, n, ins, training: bool, argmax=None):
        """One node's output from its input values; returns (y, saved) where
        saved holds the pool argmax / BatchNorm statistics backward needs."""
        op, name, a = n["op"], n["name"], n.get("attrs", {})
        x = ins[0] if ins else None
        saved = {}
        if op == "conv2d":
            s = _pair(a, "strides", 1)
            b = self.w.get(name + ".bias") if a.get("use_bias", True) else None
            co = a["filters"]
            kh, kw, ci, _ = self.w[name + ".weight"].shape
            r = (kh * kw * ci, ci, co, "fwd", kh * kw)
            y = conv2d(self._op(x, co, r), self._op(self.w[name + ".weight"], co, r), b, s,
                       a.get("padding", "valid") == "same")
        elif op == "dense":
            co = a["units"]
            r = (x.shape[1], x.shape[1], co, "fwd", 1)
            y = self._op(x, co, r) @ self._op(self.w[name + ".weight"], co, r)
            if a.get("use_bias", True):
                y = y + self.w[name + ".bias"]
        elif op == "relu":
            y = np.where(x > 0, x, 0.0)
        elif op == "gelu":
            y = gelu(x)
        elif op == "add":
            y = ins[0] + ins[1]
        elif op == "mul":
            y = ins[0] * ins[1]
        elif op == "identity":
            y = x.copy()
        elif op == "flatten":
            y = x.reshape(x.shape[0], -1)
        elif op == "max_pooling2d":
            k = _pair(a, "pool_size")
            s = _pair(a, "strides") if "strides" in a else k
            if argmax is not None:
                idx = np.asarray(argmax, dtype=np.float64)
                y = maxpool_gather(x, idx, k, s)
            else:
                y, idx = maxpool2d(x, k, s)
            saved["argmax"] = idx
        elif op == "global_avg_pool2d":
            y = avgpool(x, 1, 1)
        elif op == "batch_normalization":
            C = x.shape[-1]
            x2 = x.reshape(-1, C)
            eps = a.get("epsilon", 1e-3)
            gm, bt = self.w[name + ".gamma"], self.w[name + ".beta"]
            if training:
                mean, inv = bn_stats(x2, eps)
                saved["stats"] = (mean, inv)
            else:
                mean = self.w[name + ".moving_mean"]
                inv = 1.0 / np.sqrt(self.w[name + ".moving_variance"] + eps)
            y = (((x2 - mean) * inv) * gm + bt).reshape(x.shape)
        elif op == "layer_normalization":
            C = x.shape[-1]
            x2 = x.reshape(-1, C)
            eps = a.get("epsilon", 1e-3)
            m = x2.mean(axis=1, keepdims=True)
            var = np.maximum((x2 * x2).mean(axis=1, keepdims=True) - m * m, 0.0)
            y = ((x2 - m) / np.sqrt(var + eps) * self.w[name + ".gamma"] + self.w[name + ".beta"]).reshape(x.shape)
        else:
            raise NotImplementedError(op)
        return self._st(y), saved

    def node_vjp(self, n, ins, gy, saved):
        """Vector-Jacobian product of one node: (gradients of its inputs --
        None for graph inputs, whose gradients are dead code --, weight
        gradients)."""
        op, name, a = n["op"], n["name"], n.get("attrs", {})
        names = n.get("inputs", [])
        x = ins[0] if ins else None
        need_x = bool(names) and names[0] not in self.inputs
        gin = [None] * len(ins)
        gw = {}
        if op == "relu":
            gin[0] = np.where(x > 0, gy, 0.0)
        elif op == "gelu":
            gin[0] = gelu_grad(x, gy)
        elif op == "add":
            gin = [gy, gy]
        elif op == "mul":
            gin = [gy * ins[1], gy * ins[0]]
        elif op == "identity":
            gin[0] = gy
        elif op == "flatten":
            gin[0] = gy.reshape(x.shape)
        elif op == "dense":
            co = a["units"]
            fin = x.shape[1]
            rw, rd = (x.shape[0], fin, co, "dense_wgrad", 1), (co, co, fin, "dgrad", 1)
            gw[name + ".weight"] = self._op(x, co, rw).T @ self._op(gy, co, rw)
            if a.get("use_bias", True):
                gw[name + ".bias"] = gy.sum(axis=0)
            if need_x:
                gin[0] = self._op(gy, co, rd) @ self._op(self.w[name + ".weight"], co, rd).T
        elif op == "conv2d":
            s = _pair(a, "strides", 1)
            same = a.get("padding", "valid") == "same"
            w = self.w[name + ".weight"]
            kh, kw, ci, co = w.shape
            rw, rd = (0, ci, co, "wgrad", kh * kw), (kh * kw * co, co, ci, "dgrad", kh * kw)
            gw[name + ".weight"] = conv2d_grad_weight(self._op(x, co, rw), self._op(gy, co, rw), w.shape, s, same)
            if a.get("use_bias", True):
                gw[name + ".bias"] = gy.reshape(-1, co).sum(axis=0)
            if need_x:
                gin[0] = conv2d_grad_input(self._op(gy, co, rd), self._op(w, co, rd), x.shape, s, same)
        elif op == "max_pooling2d":
            k = _pair(a, "pool_size")
            s = _pair(a, "strides") if "strides" in a else k
            gin[0] = maxpool2d_grad(saved["argmax"], gy, x.shape, k, s)
        elif op == "global_avg_pool2d":
            gin[0] = avgpool_grad(gy, x.shape)
        elif op == "batch_normalization":
            C = x.shape[-1]
            x2, g2 = x.reshape(-1, C), gy.reshape(-1, C)
            mean, inv = saved["stats"]
            xhat = (x2 - mean) * inv
            sg, sgx = g2.sum(axis=0), (g2 * xhat).sum(axis=0)
            gw[name + ".gamma"] = sgx
            gw[name + ".beta"] = sg
            if need_x:
                M = x2.shape[0]
                gin[0] = ((self.w[name + ".gamma"] * inv) * (g2 - (sg + xhat * sgx) / M)).reshape(x.shape)
        elif op == "layer_normalization":
            C = x.shape[-1]
            x2, g2 = x.reshape(-1, C), gy.reshape(-1, C)
            eps = a.get("epsilon", 1e-3)
            m = x2.mean(axis=1, keepdims=True)
            var = np.maximum((x2 * x2).mean(axis=1, keepdims=True) - m * m, 0.0)
            rstd = 1.0 / np.sqrt(var + eps)
            xhat = (x2 - m) * rstd
            gw[name + ".gamma"] = (g2 * xhat).sum(axis=0)
            gw[name + ".beta"] = g2.sum(axis=0)
            if need_x:
                gh = g2 * self.w[name + ".gamma"]
                gin[0] = (rstd * (gh - gh.mean(axis=1, keepdims=True)
                                  - xhat * (gh * xhat).mean(axis=1, keepdims=True))).reshape(x.shape)
        else:
            raise NotImplementedError(op)
        gin = [None if (g is None or nm in self.inputs) else self._st(g) for g, nm in zip(gin, names)]
        return gin, {k: self._st(v) for k, v in gw.items()}

    # ---------------------------------------------------------------- forward
    def forward(self, feed, training: bool, argmax: Optional[Dict[str, np.ndarray]] = None):
        argmax = argmax or {}
        v = {k: self._st(np.asarray(x, dtype=np.float64)) for k, x in feed.items()}
        self.saved = {}
        self.node_saved = {}
        for n in self.nodes:
            ins = [v[i] for i in n.get("inputs", [])]
            y, sv = self.node_forward(n, ins, training, argmax.get(n["name"]))
            self.node_saved[n["name"]] = sv
            if "argmax" in sv:
                self.saved[n["name"] + ".argmax"] = sv["argmax"]
            if "stats" in sv:
                self.saved[n["name"] + ".stats"] = sv["stats"]
            v[n["name"]] = y
        self.values = v
        return {o: v[o] for o in self.outputs}

    # --------------------------------------------------------------- backward
    def loss_grad(self, out, target, loss="l1"):
        t = np.asarray(target, dtype=np.float64)
        if loss == "l1":
            lv, g = l1_loss(out, t)
        elif loss == "softmax_ce":
            lv, g = softmax_ce(out, t)
        else:
            raise ValueError(loss)
        return lv, self._st(g)

    def gradients(self, feed, target, loss: str = "l1", argmax=None):
        """Training forward, loss, reverse-mode weight gradients (float64)."""
        out = self.forward(feed, training=True, argmax=argmax)[self.outputs[0]]
        lv, gpred = self.loss_grad(out, target, loss)
        v = self.values
        grads: Dict[str, np.ndarray] = {}
        dv: Dict[str, np.ndarray] = {self.outputs[0]: gpred}
        self.value_grads = dv
        for n in reversed(self.nodes):
            gy = dv.get(n["name"])
            if gy is None:
                continue
            names = n.get("inputs", [])
            gin, gw = self.node_vjp(n, [v[i] for i in names], gy, self.node_saved[n["name"]])
            grads.update(gw)
            for nm, g in zip(names, gin):
                if g is not None:
                    dv[nm] = self._st(dv[nm] + g) if nm in dv else g
        return lv, grads


def local_forward_parity(model: "F64Model", feed, device_value, training: bool = False):
    """Launch-by-launch parity of a forward pass (inference plans: BatchNorm
    from moving statistics when training is False): every node re-evaluated
    from the device's own inputs, as local_parity's forward half. Returns
    {value: err} with err = ||dev - oracle|| / ||oracle||."""
    res = {}
    v = {k: model._st(np.asarray(x, np.float64)) for k, x in feed.items()}
    for n in model.nodes:
        name = n["name"]
        ins = [v[i] for i in n.get("inputs", [])]
        am = device_value(name + ".argmax") if n["op"] == "max_pooling2d" else None
        y, _ = model.node_forward(n, ins, training, am)
        dv = device_value(name)
        if dv is not None:
            b = np.asarray(y, np.float64)
            nb = np.linalg.norm(b)
            d = np.asarray(dv, np.float64).reshape(b.shape)
            res[name] = float(np.linalg.norm(d - b) / nb) if nb > 0 else float(np.linalg.norm(d))
            y = d
        v[name] = y
    return res


def local_parity(model: "F64Model", feed, device_value, device_grads, target, loss="l1"):
    """Launch-by-launch parity of one training step: every node is re-evaluated
    by the oracle FROM THE DEVICE'S OWN INPUTS (forward values, max-pool
    indices, BatchNorm statistics and upstream gradients read back from the
    step), so each comparison measures one kernel (or one fused group) and no
    rounding difference propagates through the depth of the network.

    device_value(name) -> array or None (None: held in fused-group registers,
    then the oracle's locally computed value stands in). Returns
    {"forward": {value: err}, "backward": {"d."+value: err}, "weights": {w: err}}
    with err = ||dev - oracle|| / ||oracle||."""
    def err(a, b):
        b = np.asarray(b, np.float64)
        nb = np.linalg.norm(b)
        return float(np.linalg.norm(np.asarray(a, np.float64).reshape(b.shape) - b) / nb) if nb > 0 else \
            float(np.linalg.norm(np.asarray(a, np.float64)))

    res = {"forward": {}, "backward": {}, "weights": {}}
    v = {k: model._st(np.asarray(x, np.float64)) for k, x in feed.items()}
    saved = {}
    for n in model.nodes:
        name = n["name"]
        ins = [v[i] for i in n.get("inputs", [])]
        am = device_value(name + ".argmax") if n["op"] == "max_pooling2d" else None
        y, sv = model.node_forward(n, ins, True, am)
        if n["op"] == "batch_normalization":
            st = device_value(name + ".stats")
            if st is not None:
                st = np.asarray(st, np.float64).reshape(2, -1)
                res["forward"][name + ".stats"] = max(err(st[0], sv["stats"][0]), err(st[1], sv["stats"][1]))
                # the device's statistics are what its apply and backward used
                sv = {"stats": (st[0], st[1])}
                C = ins[0].shape[-1]
                x2 = ins[0].reshape(-1, C)
                y = model._st((((x2 - st[0]) * st[1]) * model.w[name + ".gamma"] + model.w[name + ".beta"])
                              .reshape(ins[0].shape))
        dv = device_value(name)
        if dv is not None:
            res["forward"][name] = err(dv, y)
            y = np.asarray(dv, np.float64).reshape(y.shape)
        saved[name] = sv
        v[name] = y
    out = v[model.outputs[0]]
    _, gpred = model.loss_grad(out, target, loss)
    pred = model.outputs[0]
    g = {}
    dg = device_value("d." + pred)
    if dg is not None:
        res["backward"]["d." + pred] = err(dg, gpred)
        gpred = np.asarray(dg, np.float64).reshape(gpred.shape)
    g[pred] = gpred
    for n in reversed(model.nodes):
        name = n["name"]
        gy = g.get(name)
        if gy is None:
            continue
        if name != pred:
            dg = device_value("d." + name)
            if dg is not None:
                res["backward"]["d." + name] = err(dg, gy)
                gy = np.asarray(dg, np.float64).reshape(gy.shape)
        names = n.get("inputs", [])
        gin, gw = model.node_vjp(n, [v[i] for i in names], gy, saved[name])
        for w, gwv in gw.items():
            if w in device_grads:
                res["weights"][w] = err(device_grads[w], gwv)
        for nm, gi in zip(names, gin):
            if gi is not None:
                g[nm] = model._st(g[nm] + gi) if nm in g else gi
    return res
