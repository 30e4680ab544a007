"""oracle/reference.py -- TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/_ref/libnncref.so: the reference nnc library compiled
from /root/reference/proj sources by oracle/Makefile (namespace renamed nncref)
plus this repo's C shim oracle/ref_shim.cpp. Used by tests/ (parity checks) and
by bench.py's cpu_baseline / --impl reference legs -- never by the product.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libnncref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        # the C++ runtime must be global before an RTLD_LOCAL C++ library is
        # mapped into this (C) process, or libnncref's first std:: call faults
        ctypes.CDLL("libstdc++.so.6", mode=ctypes.RTLD_GLOBAL)
        l = ctypes.CDLL(LIB, mode=ctypes.RTLD_LOCAL)
        P, I, I64, D, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_char_p
        DP, I64P = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        for name, res, args in [
            ("ref_last_error", S, []), ("ref_model_load", P, [S, I]), ("ref_model_free", None, [P]),
            ("ref_model_describe", S, [P]), ("ref_feed", I, [P, S, DP, I64P, I]),
            ("ref_run_inference", I, [P]), ("ref_eval_all", I, [P]), ("ref_value_rank", I, [P, S, I64P]),
            ("ref_value", I, [P, S, DP, I64]), ("ref_weight", I, [P, S, DP, I64]),
            ("ref_set_weight", I, [P, S, DP, I64]), ("ref_grads", I, [P, DP, I64P, I, DP]),
            ("ref_grad", I, [P, S, DP, I64]), ("ref_train_step", I, [P, DP, I64P, I, D, DP]),
            ("ref_group_document", S, [S, I]),
            ("ref_check_partition", I, [S, I, S]),
            ("ref_init_uniform", D, [ctypes.c_uint64, S, I64, D, D]),
        ]:
            fn = getattr(l, name)
            fn.restype, fn.argtypes = res, args
        _lib = l
    return _lib


def _err():
    return lib().ref_last_error().decode()


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class RefModel:
    """The reference pipeline on one DLB document: parse_model -> optimize ->
    derive_versions -> compile_version_set(policy) -> HostModel."""

    def __init__(self, document: str, policy: int = 0):
        self.h = lib().ref_model_load(document.encode(), policy)
        if not self.h:
            raise RuntimeError("reference rejected the document: " + _err())
        self.describe = json.loads(lib().ref_model_describe(self.h).decode())
        self.weight_shapes = {k: tuple(v) for k, v in self.describe["weights"].items()}

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_model_free(self.h)
            self.h = None

    def feed(self, name, value):
        v = np.ascontiguousarray(value, dtype=np.float64)
        dims = (ctypes.c_int64 * v.ndim)(*v.shape)
        if lib().ref_feed(self.h, name.encode(), _dp(v), dims, v.ndim):
            raise RuntimeError(_err())

    def _value(self, name):
        dims = (ctypes.c_int64 * 8)()
        r = lib().ref_value_rank(self.h, name.encode(), dims)
        if r < 0:
            raise KeyError(name)
        out = np.empty(tuple(dims[:r]), dtype=np.float64)
        if lib().ref_value(self.h, name.encode(), _dp(out), out.size):
            raise RuntimeError(_err())
        return out

    def run(self, inputs, names=None):
        """runtime::execute on the inference plan; returns outputs (float64 copies)."""
        for k, v in inputs.items():
            self.feed(k, v)
        if lib().ref_run_inference(self.h):
            raise RuntimeError(_err())
        names = names or [v["name"] for v in self.describe["inference"]["values"] if v["category"] == "output"]
        return {n: self._value(n) for n in names}

    def eval_all(self, inputs, names):
        """kernels::eval_graph (REF kernels) on the optimized graph; any value by name."""
        for k, v in inputs.items():
            self.feed(k, v)
        if lib().ref_eval_all(self.h):
            raise RuntimeError(_err())
        return {n: self._value(n) for n in names}

    def weight(self, name):
        out = np.empty(self.weight_shapes[name], dtype=np.float64)
        if lib().ref_weight(self.h, name.encode(), _dp(out), out.size):
            raise RuntimeError(_err())
        return out

    def set_weight(self, name, value):
        v = np.ascontiguousarray(value, dtype=np.float64)
        if lib().ref_set_weight(self.h, name.encode(), _dp(v), v.size):
            raise RuntimeError(_err())

    def gradients(self, inputs, target):
        for k, v in inputs.items():
            self.feed(k, v)
        t = np.ascontiguousarray(target, dtype=np.float64)
        dims = (ctypes.c_int64 * t.ndim)(*t.shape)
        loss = ctypes.c_double()
        if lib().ref_grads(self.h, _dp(t), dims, t.ndim, ctypes.byref(loss)):
            raise RuntimeError(_err())
        grads = {}
        for w in self.describe["weight_grads"]:
            g = np.empty(self.weight_shapes[w], dtype=np.float64)
            if lib().ref_grad(self.h, w.encode(), _dp(g), g.size):
                raise RuntimeError(_err())
            grads[w] = g
        return loss.value, grads

    def train_step(self, inputs, target, lr):
        for k, v in inputs.items():
            self.feed(k, v)
        t = np.ascontiguousarray(target, dtype=np.float64)
        dims = (ctypes.c_int64 * t.ndim)(*t.shape)
        loss = ctypes.c_double()
        if lib().ref_train_step(self.h, _dp(t), dims, t.ndim, lr, ctypes.byref(loss)):
            raise RuntimeError(_err())
        return loss.value


def group_document(document: str, policy: int):
    res = lib().ref_group_document(document.encode(), policy)
    if res is None:
        raise RuntimeError(_err())
    return json.loads(res.decode())


def check_partition(document: str, role: int, groups) -> dict:
    """The reference harness's oracle_valid_partition / oracle_maximal_partition
    (tests/harness/oracle_groups.cpp:117-150) on one role graph
    (0 inference, 1 train_fwd, 2 train_bwd) of the document's version set."""
    r = lib().ref_check_partition(document.encode(), role, json.dumps(groups).encode())
    if r < 0:
        raise RuntimeError(_err())
    return {"valid": bool(r & 1), "maximal": bool(r & 2)}


def init_uniform(seed: int, name: str, index: int, lo: float, hi: float) -> float:
    return lib().ref_init_uniform(seed, name.encode(), index, lo, hi)
