"""oracle/restated.py -- TEST INFRASTRUCTURE ONLY.

Independent CPU oracle for DLB model documents built on the C restatement
(oracle/nnc_oracle.c -> oracle/_ref/libnnc_oracle.so): its own document walk,
its own initializer (InitStream, reference ingest.cpp:43-70), its own forward
(inference or training-mode BatchNorm) and reverse-mode gradients, L1 loss and
SGD. It covers the extension ops the reference lacks (BatchNorm, GELU,
LayerNorm): for those, parity is unpinned by the reference -- this restatement
is the oracle. For reference-vocabulary graphs it is itself checked against the
reference (tests/test_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from typing import Dict, List

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libnnc_oracle.so")
MASK = (1 << 64) - 1

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(LIB)
        _lib.o_l1_loss.restype = ctypes.c_double
    return _lib


def available() -> bool:
    return os.path.exists(LIB)


def _f(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Geom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n", "ih", "iw", "ci", "co", "kh", "kw", "sh", "sw", "oh", "ow",
                                               "pt", "pl")]


I64 = ctypes.c_int64


def conv_geom(xd, k, s, co, same):
    n, ih, iw, ci = xd
    if same:
        oh, ow = -(-ih // s[0]), -(-iw // s[1])
        pt = max((oh - 1) * s[0] + k[0] - ih, 0) // 2
        pl = max((ow - 1) * s[1] + k[1] - iw, 0) // 2
    else:
        oh, ow, pt, pl = (ih - k[0]) // s[0] + 1, (iw - k[1]) // s[1] + 1, 0, 0
    return Geom(n, ih, iw, ci, co, k[0], k[1], s[0], s[1], oh, ow, pt, pl)


def pool_params(xd, k, s):
    n, ih, iw, c = xd
    oh, ow = (ih - k[0]) // s[0] + 1, (iw - k[1]) // s[1] + 1
    return (I64 * 10)(n, ih, iw, c, k[0], k[1], s[0], s[1], oh, ow), (n, oh, ow, c)


def empty(shape):
    return np.zeros(shape, dtype=np.float32)


# --------------------------------------------------------------------------
# deterministic initializer (restated InitStream, reference ingest.cpp:43-70)
# --------------------------------------------------------------------------

def fnv1a64(text: str) -> int:
    h = 14695981039346656037
    for c in text.encode():
        h = ((h ^ c) * 1099511628211) & MASK
    return h


def init_uniform(seed: int, name: str, n: int, lo: float, hi: float) -> np.ndarray:
    s = (seed ^ fnv1a64(name)) & MASK
    s = (s * 6364136223846793005 + 1442695040888963407) & MASK
    out = np.empty(n, dtype=np.float64)
    for i in range(n):
        s = (s * 6364136223846793005 + 1442695040888963407) & MASK
        out[i] = lo + ((s >> 11) * 2.0 ** -53) * (hi - lo)
    return out


def init_weight(seed, name, shape, fan_in):
    b = 1.0 / math.sqrt(fan_in)
    return init_uniform(seed, name, int(np.prod(shape)), -b, b).astype(np.float32).reshape(shape)


def _pair(a, key, default=None):
    v = a.get(key, default)
    return (v, v) if isinstance(v, int) else tuple(v)


class OracleModel:
    """A DLB document evaluated by the restated kernels."""

    def __init__(self, document: str, weights: Dict[str, np.ndarray] | None = None):
        d = json.loads(document)
        self.seed = d.get("seed", 0)
        self.nodes = d["nodes"]
        self.outputs = d["outputs"]
        self.inputs = {i["name"]: tuple(i["shape"]) for i in d["inputs"]}
        self.w: Dict[str, np.ndarray] = {}
        dims = dict(self.inputs)
        for n in self.nodes:
            op, name, a = n["op"], n["name"], n.get("attrs", {})
            x = dims[n["inputs"][0]] if n.get("inputs") else None
            if op == "conv2d":
                k, s = _pair(a, "kernel_size"), _pair(a, "strides", 1)
                co = a["filters"]
                self.w[name + ".weight"] = init_weight(self.seed, name + ".weight", (k[0], k[1], x[3], co),
                                                       k[0] * k[1] * x[3])
                if a.get("use_bias", True):
                    self.w[name + ".bias"] = init_weight(self.seed, name + ".bias", (co,), k[0] * k[1] * x[3])
                g = conv_geom(x, k, s, co, a.get("padding", "valid") == "same")
                dims[name] = (g.n, g.oh, g.ow, co)
            elif op == "dense":
                u = a["units"]
                self.w[name + ".weight"] = init_weight(self.seed, name + ".weight", (x[1], u), x[1])
                if a.get("use_bias", True):
                    self.w[name + ".bias"] = init_weight(self.seed, name + ".bias", (u,), x[1])
                dims[name] = (x[0], u)
            elif op == "max_pooling2d":
                k = _pair(a, "pool_size")
                s = _pair(a, "strides", k[0]) if "strides" in a else k
                dims[name] = pool_params(x, k, s)[1]
            elif op == "global_avg_pool2d":
                dims[name] = (x[0], 1, 1, x[3])
            elif op == "flatten":
                dims[name] = (x[0], int(np.prod(x[1:])))
            elif op in ("batch_normalization", "layer_normalization"):
                c = x[-1]
                self.w[name + ".gamma"] = np.ones(c, np.float32)
                self.w[name + ".beta"] = np.zeros(c, np.float32)
                if op == "batch_normalization":
                    self.w[name + ".moving_mean"] = np.zeros(c, np.float32)
                    self.w[name + ".moving_variance"] = np.ones(c, np.float32)
                dims[name] = x
            else:
                dims[name] = x
        self.dims = dims
        if weights:
            for k, v in weights.items():
                self.w[k] = np.ascontiguousarray(v, dtype=np.float32)

    # ---------------------------------------------------------------- forward
    def forward(self, feed: Dict[str, np.ndarray], training: bool):
        L = lib()
        v = {k: np.ascontiguousarray(x, dtype=np.float32) for k, x in feed.items()}
        self.saved = {}
        for n in self.nodes:
            op, name, a = n["op"], n["name"], n.get("attrs", {})
            ins = [v[i] for i in n.get("inputs", [])]
            x = ins[0] if ins else None
            if op == "conv2d":
                k, s = _pair(a, "kernel_size"), _pair(a, "strides", 1)
                g = conv_geom(x.shape, k, s, a["filters"], a.get("padding", "valid") == "same")
                y = empty((g.n, g.oh, g.ow, g.co))
                b = self.w.get(name + ".bias") if a.get("use_bias", True) else None
                L.o_conv2d(_f(x), _f(self.w[name + ".weight"]), _f(b) if b is not None else None, _f(y),
                           ctypes.byref(g))
            elif op == "dense":
                y = empty((x.shape[0], a["units"]))
                b = self.w.get(name + ".bias") if a.get("use_bias", True) else None
                L.o_dense(_f(x), _f(self.w[name + ".weight"]), _f(b) if b is not None else None, _f(y),
                          I64(x.shape[0]), I64(x.shape[1]), I64(a["units"]))
            elif op == "relu":
                y = empty(x.shape)
                L.o_relu(_f(x), _f(y), I64(x.size))
            elif op == "gelu":
                y = empty(x.shape)
                L.o_gelu(_f(x), _f(y), I64(x.size))
            elif op in ("add", "mul"):
                y = empty(x.shape)
                getattr(L, "o_" + op)(_f(ins[0]), _f(ins[1]), _f(y), I64(x.size))
            elif op in ("identity",):
                y = x.copy()
            elif op == "flatten":
                y = x.reshape(x.shape[0], -1).copy()
            elif op == "max_pooling2d":
                k = _pair(a, "pool_size")
                s = _pair(a, "strides", k[0]) if "strides" in a else k
                pp, oshape = pool_params(x.shape, k, s)
                y, idx = empty(oshape), empty(oshape)
                L.o_maxpool2d(_f(x), _f(y), _f(idx), pp)
                self.saved[name + ".argmax"] = idx
            elif op == "global_avg_pool2d":
                y = empty((x.shape[0], 1, 1, x.shape[3]))
                L.o_avgpool(_f(x), _f(y), *[I64(t) for t in (x.shape[0], x.shape[1], x.shape[2], x.shape[3], 1, 1)])
            elif op == "batch_normalization":
                C = x.shape[-1]
                rows = x.size // C
                y = empty(x.shape)
                eps = ctypes.c_double(a.get("epsilon", 1e-3))
                gm, bt = self.w[name + ".gamma"], self.w[name + ".beta"]
                if training:
                    st = empty((2, C))
                    L.o_bn_stats(_f(x), _f(st), I64(rows), I64(C), eps)
                    L.o_bn_apply(_f(x), _f(st), _f(gm), _f(bt), _f(y), I64(rows), I64(C))
                    self.saved[name + ".stats"] = st
                else:
                    L.o_bn_infer(_f(x), _f(self.w[name + ".moving_mean"]), _f(self.w[name + ".moving_variance"]),
                                 _f(gm), _f(bt), _f(y), I64(rows), I64(C), eps)
            elif op == "layer_normalization":
                C = x.shape[-1]
                y = empty(x.shape)
                L.o_layernorm(_f(x), _f(self.w[name + ".gamma"]), _f(self.w[name + ".beta"]), _f(y),
                              I64(x.size // C), I64(C), ctypes.c_double(a.get("epsilon", 1e-3)))
            else:
                raise NotImplementedError(op)
            v[name] = y
        self.values = v
        return {o: v[o] for o in self.outputs}

    # --------------------------------------------------------------- backward
    def gradients(self, feed, target):
        """Training forward, L1 loss (runtime.cpp:468-483), reverse-mode weight gradients."""
        L = lib()
        out = self.forward(feed, training=True)[self.outputs[0]]
        t = np.ascontiguousarray(target, dtype=np.float32)
        gpred = empty(out.shape)
        loss = L.o_l1_loss(_f(out), _f(t), _f(gpred), I64(out.size))
        v = self.values
        grads: Dict[str, np.ndarray] = {}
        dv: Dict[str, List[np.ndarray]] = {self.outputs[0]: [gpred]}

        def acc(name, g):
            dv.setdefault(name, []).append(g)

        def total(name):
            lst = dv.get(name)
            if not lst:
                return None
            s = lst[0]
            for g in lst[1:]:
                r = empty(s.shape)
                L.o_add(_f(s), _f(g), _f(r), I64(s.size))
                s = r
            return s

        for n in reversed(self.nodes):
            op, name, a = n["op"], n["name"], n.get("attrs", {})
            gy = total(name)
            if gy is None:
                continue
            ins = n.get("inputs", [])
            x = v[ins[0]] if ins else None
            if op == "relu":
                gx = empty(x.shape)
                L.o_relu_grad(_f(x), _f(gy), _f(gx), I64(x.size))
                acc(ins[0], gx)
            elif op == "gelu":
                gx = empty(x.shape)
                L.o_gelu_grad(_f(x), _f(gy), _f(gx), I64(x.size))
                acc(ins[0], gx)
            elif op == "add":
                acc(ins[0], gy)
                acc(ins[1], gy)
            elif op == "mul":
                ga, gb = empty(x.shape), empty(x.shape)
                L.o_mul(_f(gy), _f(v[ins[1]]), _f(ga), I64(x.size))
                L.o_mul(_f(gy), _f(v[ins[0]]), _f(gb), I64(x.size))
                acc(ins[0], ga)
                acc(ins[1], gb)
            elif op == "identity":
                acc(ins[0], gy)
            elif op == "flatten":
                acc(ins[0], gy.reshape(x.shape).copy())
            elif op == "dense":
                B, I, O = x.shape[0], x.shape[1], a["units"]
                gw = empty((I, O))
                L.o_dense_grad_weight(_f(x), _f(gy), _f(gw), I64(B), I64(I), I64(O))
                grads[name + ".weight"] = gw
                if a.get("use_bias", True):
                    gb = empty((O,))
                    L.o_sum_cols(_f(gy), _f(gb), I64(B), I64(O))
                    grads[name + ".bias"] = gb
                if ins[0] not in self.inputs:
                    gx = empty(x.shape)
                    L.o_dense_grad_input(_f(gy), _f(self.w[name + ".weight"]), _f(gx), I64(B), I64(I), I64(O))
                    acc(ins[0], gx)
            elif op == "conv2d":
                k, s = _pair(a, "kernel_size"), _pair(a, "strides", 1)
                g = conv_geom(x.shape, k, s, a["filters"], a.get("padding", "valid") == "same")
                gw = empty((k[0], k[1], x.shape[3], a["filters"]))
                L.o_conv2d_grad_weight(_f(x), _f(gy), _f(gw), ctypes.byref(g))
                grads[name + ".weight"] = gw
                if a.get("use_bias", True):
                    gb = empty((a["filters"],))
                    L.o_sum_nhw(_f(gy), _f(gb), I64(gy.size // a["filters"]), I64(a["filters"]))
                    grads[name + ".bias"] = gb
                if ins[0] not in self.inputs:
                    gx = empty(x.shape)
                    L.o_conv2d_grad_input(_f(gy), _f(self.w[name + ".weight"]), _f(gx), ctypes.byref(g))
                    acc(ins[0], gx)
            elif op == "max_pooling2d":
                k = _pair(a, "pool_size")
                s = _pair(a, "strides", k[0]) if "strides" in a else k
                pp, _ = pool_params(x.shape, k, s)
                gx = empty(x.shape)
                L.o_maxpool2d_grad(_f(self.saved[name + ".argmax"]), _f(gy), _f(gx), pp)
                acc(ins[0], gx)
            elif op == "global_avg_pool2d":
                gx = empty(x.shape)
                L.o_avgpool_grad(_f(gy), _f(gx), *[I64(t) for t in (x.shape[0], x.shape[1], x.shape[2], x.shape[3], 1, 1)])
                acc(ins[0], gx)
            elif op == "batch_normalization":
                C = x.shape[-1]
                rows = x.size // C
                st = self.saved[name + ".stats"]
                sg, sgx = empty((C,)), empty((C,))
                L.o_bn_grad_reduce(_f(x), _f(st), _f(gy), _f(sg), _f(sgx), I64(rows), I64(C))
                grads[name + ".gamma"] = sgx
                grads[name + ".beta"] = sg
                if ins[0] not in self.inputs:
                    gx = empty(x.shape)
                    L.o_bn_grad_input(_f(x), _f(st), _f(gy), _f(self.w[name + ".gamma"]), _f(sg), _f(sgx), _f(gx),
                                      I64(rows), I64(C))
                    acc(ins[0], gx)
            elif op == "layer_normalization":
                C = x.shape[-1]
                rows = x.size // C
                eps = ctypes.c_double(a.get("epsilon", 1e-3))
                dg, db = empty((C,)), empty((C,))
                L.o_layernorm_dgamma(_f(x), _f(gy), _f(dg), I64(rows), I64(C), eps)
                L.o_sum_cols(_f(gy), _f(db), I64(rows), I64(C))
                grads[name + ".gamma"] = dg
                grads[name + ".beta"] = db
                if ins[0] not in self.inputs:
                    gx = empty(x.shape)
                    L.o_layernorm_grad_input(_f(x), _f(self.w[name + ".gamma"]), _f(gy), _f(gx), I64(rows), I64(C),
                                             eps)
                    acc(ins[0], gx)
            else:
                raise NotImplementedError(op)
        return loss, grads
