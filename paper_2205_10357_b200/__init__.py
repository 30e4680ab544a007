"""paper_2205_10357_b200 -- B200-native execution backend for SOL-style compiled networks.

Python mirror of the reference's C++ pipeline (nnc::ingest / passes / autodiff /
plan / runtime), bound through the C-ABI in include/nnc_b200.h. The compute path
is libnnc_b200.so (C++ host: partitioning, buffer planning, launch scheduling)
over libnncb.so (hand-written sm_100a kernels, include/nncb.h). There is no CPU
fallback: the native libraries are loaded on first use (so importing the
package's pure-Python helpers, e.g. `workloads`, maps no native code), and
that first use raises if they are missing.

Reference call chain being replaced (file:line in /root/reference/proj):
    ingest::parse_model        core/src/ingest.cpp:411-500
    passes::optimize           core/src/passes.cpp:785-793
    autodiff::derive_versions  core/src/autodiff.cpp:89-319
    plan::compile_version_set  core/src/plan.cpp:441-457
    runtime::execute           core/src/runtime.cpp:314-462
    runtime::train_step        core/src/runtime.cpp:498-537
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
HOST_LIB = os.path.join(LIB_DIR, "libnnc_b200.so")
KERNEL_LIB = os.path.join(LIB_DIR, "libnncb.so")

PREC_TF32 = 0   # tcgen05.mma kind::tf32, fp32 accumulation in TMEM
PREC_FP32 = 1   # exact-order fp32 (bit-identical to the reference CPU kernels)
PREC_BF16 = 2   # tcgen05.mma kind::f16 on bf16 operand copies for the forward / input-gradient
                # contractions (K-major operands), fp32 accumulate; weight gradients tf32
PREC_TF32X3 = 3  # fp32-grade tensor-core path: operands split into tf32 hi + lo parts,
                 # kind::tf32 over the K-concatenated problem (A_hi B_hi + A_hi B_lo + A_lo B_hi)


class NNCError(RuntimeError):
    """Mirror of nnc::Error: `code` is the reference Error::Code value (error.hpp:12-31)."""

    CODES = ["UnknownOp", "ShapeMismatch", "MissingSeed", "BadMagic", "TruncatedTensor",
             "DuplicateName", "RankError", "ExtentMismatch", "UnknownSymbol", "IllegalOverride",
             "NoBackend", "UnsupportedInGroup", "NonDifferentiable", "UnboundVdim",
             "ArenaOverflow", "MissingGrad", "BadToken", "BadDocument", "DeviceError"]

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = self.CODES[status - 1] if 1 <= status <= len(self.CODES) else "Internal"
        super().__init__(f"{self.code}: {message}")


def _load():
    if not os.path.exists(HOST_LIB):
        raise ImportError(f"{HOST_LIB} is not built; run __graft_entry__.build()")
    kern = ctypes.CDLL(KERNEL_LIB, mode=ctypes.RTLD_GLOBAL)
    host = ctypes.CDLL(HOST_LIB, mode=ctypes.RTLD_GLOBAL)
    P, I, I64, D, U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
    FP, I64P, DP, S = (ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64),
                       ctypes.POINTER(ctypes.c_double), ctypes.c_char_p)
    sig = {
        "nnc_last_error": (S, []),
        "nnc_last_status": (I, []),
        "nnc_model_compile": (P, [S, I]),
        "nnc_model_compile_ex": (P, [S, I, ctypes.POINTER(ctypes.c_int32), I]),
        "nnc_model_output_dims": (I, [P, S, I64P, ctypes.POINTER(ctypes.c_int)]),
        "nnc_model_free": (None, [P]),
        "nnc_model_describe": (S, [P]),
        "nnc_model_set_weight": (I, [P, S, FP, I64]),
        "nnc_model_get_weight": (I, [P, S, FP, I64]),
        "nnc_model_set_input": (I, [P, S, FP, I64P, I]),
        "nnc_model_run": (I, [P, I]),
        "nnc_model_output": (I, [P, S, FP, I64]),
        "nnc_model_train_step": (I, [P, FP, I64, D, DP]),
        "nnc_model_stage_step": (I, [P, FP, I64]),
        "nnc_model_stage_run": (I, [P, I]),
        "nnc_model_run_staged": (I, [P, I, S]),
        "nnc_model_staged_outputs": (I, [P, I]),
        "nnc_model_train_step_staged": (I, [P, D]),
        "nnc_model_staged_loss": (I, [P, DP]),
        "nnc_model_gradients": (I, [P, FP, I64, DP]),
        "nnc_model_grad": (I, [P, S, FP, I64]),
        "nnc_model_debug_keep_values": (I, [P, I]),
        "nnc_model_set_loss": (I, [P, I]),
        "nnc_model_trainer_value": (I, [P, S, FP, I64, I64P, ctypes.POINTER(ctypes.c_int)]),
        "nnc_model_run_value": (I, [P, I, S, FP, I64, I64P, ctypes.POINTER(ctypes.c_int)]),
        "nnc_model_trainer_prepare": (I, [P, FP, I64]),
        "nnc_model_trainer_step_device": (I, [P, D]),
        "nnc_model_trainer_loss": (I, [P, DP]),
        "nnc_model_launches_per_step": (U64, [P]),
        "nnc_model_profile_step": (S, [P, D]),
        "nnc_model_profile_run": (S, [P, I]),
        "nnc_model_tune": (S, [P, I, I, S]),
        "nnc_model_dp_schedule": (S, [P, I64]),
        "nnc_model_step_schedule": (S, [P, I64, I, I]),
        "nnc_model_arena_bytes": (U64, [P]),
        "nnc_model_infer_device": (I, [P]),
        "nnc_model_run_device": (I, [P, I]),
        "nnc_model_save_plans": (I, [P, ctypes.c_char_p, U64, ctypes.POINTER(ctypes.c_uint64)]),
        "nnc_model_load_plans": (I, [P, ctypes.c_char_p, U64]),
        "nnc_model_memory": (I, [P, I, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                                 ctypes.POINTER(ctypes.c_uint64)]),
        "nnc_device_sync_stats": (I, [I, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.POINTER(ctypes.c_uint64)]),
        "nnc_model_run_outputs": (I, [P, I, ctypes.c_char_p]),
        "nnc_model_set_input_borrowed": (I, [P, ctypes.c_char_p, ctypes.POINTER(ctypes.c_float),
                                             ctypes.POINTER(ctypes.c_int64), I]),
        "nnc_device_ctx": (P, []),
        "nnc_model_check_kernels": (I, [P]),
        "nnc_comm_unique_id": (I, [ctypes.c_char_p]),
        "nnc_init_comm": (I, [I, I, ctypes.c_char_p]),
        "nnc_group_document": (S, [S, S]),
        "nnc_group_document_role": (S, [S, I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(host, name)
        fn.restype, fn.argtypes = res, args
    ksig = {
        "nncb_last_error": (S, []),
        "nncb_event_create": (I, [ctypes.POINTER(P)]),
        "nncb_event_record": (I, [P, P]),
        "nncb_event_elapsed_ms": (I, [P, P, ctypes.POINTER(ctypes.c_float)]),
        "nncb_event_destroy": (I, [P]),
        "nncb_sync": (I, [P]),
        "nncb_launch_count": (U64, [P]),
    }
    for name, (res, args) in ksig.items():
        fn = getattr(kern, name)
        fn.restype, fn.argtypes = res, args
    return host, kern


_libs = None


def _lib_pair():
    global _libs
    if _libs is None:
        _libs = _load()
    return _libs


class _LazyLib:
    """Attribute access loads libnncb.so / libnnc_b200.so on first use."""

    def __init__(self, index: int):
        self._index = index

    def __getattr__(self, name):
        return getattr(_lib_pair()[self._index], name)


_host, _kern = _LazyLib(0), _LazyLib(1)


def load_native():
    """Load the native libraries now (raises ImportError if they are not built)."""
    _lib_pair()


def _check(status: int):
    if status != 0:
        raise NNCError(status, _host.nnc_last_error().decode())


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def group_document(document: str, assignment: Optional[Dict[str, int]] = None):
    """backends::group_layers on the optimized inference graph of a DLB document."""
    res = _host.nnc_group_document(document.encode(),
                                   json.dumps(assignment).encode() if assignment is not None else None)
    if res is None:
        raise NNCError(_host.nnc_last_status(), _host.nnc_last_error().decode())
    return json.loads(res.decode())


def group_document_role(document: str, role: str = "train_bwd"):
    """The B200 partition (backends::group_layers, default assignment) of one
    role graph of the document's version set: [{"backend", "members"}]."""
    r = {"inference": 0, "train_fwd": 1, "train_bwd": 2}[role]
    res = _host.nnc_group_document_role(document.encode(), r)
    if res is None:
        raise NNCError(_host.nnc_last_status(), _host.nnc_last_error().decode())
    return json.loads(res.decode())


class CompiledModel:
    """A document compiled through optimize -> derive_versions -> compile_version_set,
    holding its HostModel (weights + stamps) on the B200 runtime."""

    def __init__(self, document: str, precision: int = PREC_TF32, dynamic_vdims: Sequence[int] = (),
                 loss: str = "l1"):
        """dynamic_vdims: free vdims (#k) of the document to enable
        (passes::VdimBinding::enable) -- e.g. (0,) for a dynamic batch.
        loss: "l1" (the reference's) or "softmax_ce" (targets are probability rows)."""
        ids = (ctypes.c_int32 * max(len(dynamic_vdims), 1))(*dynamic_vdims)
        h = _host.nnc_model_compile_ex(document.encode(), precision, ids, len(dynamic_vdims))
        if not h:
            raise NNCError(_host.nnc_last_status(), _host.nnc_last_error().decode())
        self._h = h
        if loss != "l1":
            _check(_host.nnc_model_set_loss(h, {"l1": 0, "softmax_ce": 1}[loss]))
        self.describe = json.loads(_host.nnc_model_describe(h).decode())
        self.weight_shapes = {k: tuple(v) for k, v in self.describe["weights"].items()}
        inf = self.describe["inference"]
        outs = [v for v in inf["values"] if v["category"] == "output"]
        self.pred = outs[0]["name"] if outs else None

    def __del__(self):
        if getattr(self, "_h", None):
            _host.nnc_model_free(self._h)
            self._h = None

    # -- weights (HostModel) --------------------------------------------
    def weight(self, name: str) -> np.ndarray:
        out = np.empty(self.weight_shapes[name], dtype=np.float32)
        _check(_host.nnc_model_get_weight(self._h, name.encode(), _fptr(out), out.size))
        return out

    def set_weight(self, name: str, value: np.ndarray):
        v = np.ascontiguousarray(value, dtype=np.float32)
        _check(_host.nnc_model_set_weight(self._h, name.encode(), _fptr(v), v.size))

    # -- execution --------------------------------------------------------
    def feed(self, name: str, value: np.ndarray):
        v = np.ascontiguousarray(value, dtype=np.float32)
        dims = (ctypes.c_int64 * v.ndim)(*v.shape)
        _check(_host.nnc_model_set_input(self._h, name.encode(), _fptr(v), dims, v.ndim))

    def _borrow(self, inputs: Dict[str, np.ndarray]):
        """Feed inputs without a host copy; returns the arrays that must stay
        alive until the consuming call returns."""
        keep = []
        for k, v in inputs.items():
            a = np.ascontiguousarray(v, dtype=np.float32)
            keep.append(a)
            dims = (ctypes.c_int64 * a.ndim)(*a.shape)
            _check(_host.nnc_model_set_input_borrowed(self._h, k.encode(), _fptr(a), dims, a.ndim))
        return keep

    def _plan_value(self, role: str, name: str):
        for v in self.describe[role]["values"]:
            if v["name"] == name:
                return v
        raise KeyError(name)

    def run(self, inputs: Dict[str, np.ndarray], role: str = "inference",
            outputs: Optional[Sequence[str]] = None) -> Dict[str, np.ndarray]:
        """runtime::execute on the inference (or train_fwd) plan; returns every output,
        or only `outputs` (the others stay on the device)."""
        keep = self._borrow(inputs)   # noqa: F841  (alive until the run returns)
        r = 1 if role == "train_fwd" else 0
        if outputs is None:
            _check(_host.nnc_model_run(self._h, r))
        else:
            _check(_host.nnc_model_run_outputs(self._h, r, ",".join(outputs).encode()))
        out = {}
        plan = self.describe[role]
        out_names = [plan["values"][i]["name"] for i in range(len(plan["values"]))
                     if plan["values"][i]["category"] in ("output", "saved") and plan["values"][i]["resident"]]
        if outputs is not None:
            out_names = [n for n in out_names if n in set(outputs)]
        for name in out_names:
            v = self._plan_value(role, name)
            if v["storage"] != "buffer":
                continue
            dims = (ctypes.c_int64 * 8)()
            rank = ctypes.c_int()
            if _host.nnc_model_output_dims(self._h, name.encode(), dims, ctypes.byref(rank)) != 0:
                continue
            arr = np.empty(tuple(dims[: rank.value]), dtype=np.float32)
            if _host.nnc_model_output(self._h, name.encode(), _fptr(arr), arr.size) == 0:
                out[name] = arr
        return out

    def _collect(self, role: str, outputs: Optional[Sequence[str]]) -> Dict[str, np.ndarray]:
        out = {}
        plan = self.describe[role]
        out_names = [v["name"] for v in plan["values"] if v["category"] in ("output", "saved") and v["resident"]]
        if outputs is not None:
            out_names = [n for n in out_names if n in set(outputs)]
        for name in out_names:
            v = self._plan_value(role, name)
            if v["storage"] != "buffer":
                continue
            arr = np.empty(v["dims"], dtype=np.float32)
            if _host.nnc_model_output(self._h, name.encode(), _fptr(arr), arr.size) == 0:
                out[name] = arr
        return out

    def run_many(self, batches, role: str = "inference",
                 outputs: Optional[Sequence[str]] = None) -> List[Dict[str, np.ndarray]]:
        """run() over an iterable of input dicts from host buffers, returning
        each run's outputs; the upload of run i + 1 overlaps run i."""
        r = 1 if role == "train_fwd" else 0
        names = ",".join(outputs).encode() if outputs is not None else b""
        it = iter(batches)
        results: List[Dict[str, np.ndarray]] = []
        first = next(it, None)
        if first is None:
            return results
        keep = self._borrow(first)   # noqa: F841
        _check(_host.nnc_model_stage_run(self._h, r))
        pending = next(it, None)
        while True:
            _check(_host.nnc_model_run_staged(self._h, r, names))
            staged_next = pending is not None
            if staged_next:
                keep = self._borrow(pending)   # noqa: F841  (consumed by the stage call)
                _check(_host.nnc_model_stage_run(self._h, r))
                pending = next(it, None)
            _check(_host.nnc_model_staged_outputs(self._h, r))
            results.append(self._collect(role, outputs))
            if not staged_next:
                return results

    def train_step(self, inputs: Dict[str, np.ndarray], target: np.ndarray, lr: float) -> float:
        keep = self._borrow(inputs)   # noqa: F841
        t = np.ascontiguousarray(target, dtype=np.float32)
        loss = ctypes.c_double()
        _check(_host.nnc_model_train_step(self._h, _fptr(t), t.size, lr, ctypes.byref(loss)))
        return loss.value

    def train_steps(self, batches, lr: float) -> List[float]:
        """One training step per (inputs, target) pair of `batches` (any
        iterable), from host buffers, returning each step's loss. The upload of
        step i + 1 runs on the copy stream while step i computes; each step's
        result equals train_step's."""
        it = iter(batches)
        losses: List[float] = []
        first = next(it, None)
        if first is None:
            return losses
        self._stage(*first)
        pending = next(it, None)   # the step after the one being launched
        loss = ctypes.c_double()
        while True:
            _check(_host.nnc_model_train_step_staged(self._h, lr))
            staged_next = pending is not None
            if staged_next:
                self._stage(*pending)   # uploads while the launched step computes
                pending = next(it, None)
            _check(_host.nnc_model_staged_loss(self._h, ctypes.byref(loss)))
            losses.append(loss.value)
            if not staged_next:
                return losses

    def _stage(self, inputs: Dict[str, np.ndarray], target: np.ndarray):
        keep = self._borrow(inputs)   # noqa: F841  (host bytes are consumed before the call returns)
        t = np.ascontiguousarray(target, dtype=np.float32)
        _check(_host.nnc_model_stage_step(self._h, _fptr(t), t.size))

    def gradients(self, inputs: Dict[str, np.ndarray], target: np.ndarray):
        keep = self._borrow(inputs)   # noqa: F841
        t = np.ascontiguousarray(target, dtype=np.float32)
        loss = ctypes.c_double()
        _check(_host.nnc_model_gradients(self._h, _fptr(t), t.size, ctypes.byref(loss)))
        grads = {}
        for w in self.describe["weight_grads"]:
            g = np.empty(self.weight_shapes[w], dtype=np.float32)
            _check(_host.nnc_model_grad(self._h, w.encode(), _fptr(g), g.size))
            grads[w] = g
        return loss.value, grads

    # -- parity debugging ---------------------------------------------------
    def debug_keep_values(self, on: bool = True):
        """Bind the training step without arena reuse so every value survives
        the step (then read them with step_value)."""
        _check(_host.nnc_model_debug_keep_values(self._h, 1 if on else 0))

    def run_value(self, name: str, role: str = "inference") -> np.ndarray:
        """A value of the last run() (debug_keep_values(True) first): launch-by-launch
        parity of inference plans."""
        r = 1 if role == "train_fwd" else 0
        dims = (ctypes.c_int64 * 8)()
        rank = ctypes.c_int()
        _check(_host.nnc_model_run_value(self._h, r, name.encode(), None, 0, dims, ctypes.byref(rank)))
        arr = np.empty(tuple(dims[: rank.value]), dtype=np.float32)
        _check(_host.nnc_model_run_value(self._h, r, name.encode(), _fptr(arr), arr.size, dims, ctypes.byref(rank)))
        return arr

    def step_value(self, name: str) -> np.ndarray:
        """Device contents of a value of the last training step (forward or
        backward); raises NNCError for values held in fused-group registers."""
        dims = (ctypes.c_int64 * 8)()
        rank = ctypes.c_int()
        _check(_host.nnc_model_trainer_value(self._h, name.encode(), None, 0, dims, ctypes.byref(rank)))
        out = np.empty(tuple(dims[: rank.value]), dtype=np.float32)
        _check(_host.nnc_model_trainer_value(self._h, name.encode(), _fptr(out), out.size, dims, ctypes.byref(rank)))
        return out

    # -- device-resident stepping (benchmarks) ------------------------------
    def trainer_prepare(self, inputs: Dict[str, np.ndarray], target: np.ndarray):
        keep = self._borrow(inputs)   # noqa: F841
        t = np.ascontiguousarray(target, dtype=np.float32)
        _check(_host.nnc_model_trainer_prepare(self._h, _fptr(t), t.size))

    def trainer_step_device(self, lr: float):
        _check(_host.nnc_model_trainer_step_device(self._h, lr))

    def trainer_loss(self) -> float:
        loss = ctypes.c_double()
        _check(_host.nnc_model_trainer_loss(self._h, ctypes.byref(loss)))
        return loss.value

    def profile_step(self, lr: float = 0.0):
        """Per-launch device times of one eager training step (CUDA events)."""
        res = _host.nnc_model_profile_step(self._h, lr)
        if res is None:
            raise NNCError(100, _host.nnc_last_error().decode())
        return json.loads(res.decode())

    def profile_run(self, inputs: Dict[str, np.ndarray], role: str = "inference"):
        """Per-launch device times of one eager run of a plan (CUDA events)."""
        keep = self._borrow(inputs)   # noqa: F841
        res = _host.nnc_model_profile_run(self._h, 1 if role == "train_fwd" else 0)
        if res is None:
            raise NNCError(100, _host.nnc_last_error().decode())
        return json.loads(res.decode())

    def tune(self, warmup: int = 1, trials: int = 5, injected: Optional[dict] = None) -> dict:
        """Measured layer-wise tuning (backends::tune_with_report) of the three
        role graphs before first execution; the chosen GEMM tiles are attached
        to the plans (and saved with them). `injected` = {node: {"b200_gemm" |
        "b200_fused": cost}} skips the device. Returns the report."""
        inj = json.dumps(injected).encode() if injected is not None else None
        res = _host.nnc_model_tune(self._h, warmup, trials, inj)
        if res is None:
            raise NNCError(_host.nnc_last_status(), _host.nnc_last_error().decode())
        report = json.loads(res.decode())
        self.describe = json.loads(_host.nnc_model_describe(self._h).decode())   # plans now carry tiles
        return report

    def dp_schedule(self, bucket_bytes: int = 32 << 20) -> dict:
        """Data-parallel region layout and all-reduce bucket schedule (host-only)."""
        res = _host.nnc_model_dp_schedule(self._h, bucket_bytes)
        if res is None:
            raise NNCError(100, _host.nnc_last_error().decode())
        return json.loads(res.decode())

    def step_schedule(self, bucket_bytes: int = 32 << 20, comm: bool = True, sgd: bool = True) -> dict:
        """The backward half of the training step as the Trainer issues it
        (forks, per-bucket all-reduces and updates, join) -- host-only."""
        res = _host.nnc_model_step_schedule(self._h, bucket_bytes, 1 if comm else 0, 1 if sgd else 0)
        if res is None:
            raise NNCError(100, _host.nnc_last_error().decode())
        return json.loads(res.decode())

    def launches_per_step(self) -> int:
        return int(_host.nnc_model_launches_per_step(self._h))

    def save_plans(self) -> bytes:
        """SOLP bytes of the compiled plans (deterministic)."""
        n = ctypes.c_uint64()
        _check(_host.nnc_model_save_plans(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(_host.nnc_model_save_plans(self._h, buf, n.value, ctypes.byref(n)))
        return buf.raw[: n.value]

    def load_plans(self, data: bytes):
        """Replace the compiled plans with a SOLP stream (deploy path)."""
        _check(_host.nnc_model_load_plans(self._h, data, len(data)))
        self.describe = json.loads(_host.nnc_model_describe(self._h).decode())

    def memory(self, role: str = "training") -> Dict[str, int]:
        """Bound program memory vs the static planner (arena span, live high water, estimate)."""
        a, lh, e = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        r = {"inference": 0, "train_fwd": 1, "training": 2}[role]
        _check(_host.nnc_model_memory(self._h, r, ctypes.byref(a), ctypes.byref(lh), ctypes.byref(e)))
        return {"arena_bytes": a.value, "live_high_water": lh.value, "estimate": e.value}

    def arena_bytes(self) -> int:
        return int(_host.nnc_model_arena_bytes(self._h))

    def check_kernels(self):
        """NVRTC-compile every generated fused-group kernel (no GPU needed)."""
        _check(_host.nnc_model_check_kernels(self._h))

    def infer_device(self):
        _check(_host.nnc_model_infer_device(self._h))

    def run_device(self, role: str = "inference"):
        """Replay `role` with inputs already resident (from the last run() of that role)."""
        _check(_host.nnc_model_run_device(self._h, 1 if role == "train_fwd" else 0))


class DeviceTimer:
    """CUDA events on the runtime's compute stream (the stream every kernel of
    the backend is launched on)."""

    def __init__(self):
        self.ctx = _host.nnc_device_ctx()
        if not self.ctx:
            raise NNCError(100, _host.nnc_last_error().decode())
        self.a, self.b = ctypes.c_void_p(), ctypes.c_void_p()
        _kern.nncb_event_create(ctypes.byref(self.a))
        _kern.nncb_event_create(ctypes.byref(self.b))

    def start(self):
        _kern.nncb_event_record(self.ctx, self.a)

    def stop(self) -> float:
        _kern.nncb_event_record(self.ctx, self.b)
        ms = ctypes.c_float()
        if _kern.nncb_event_elapsed_ms(self.a, self.b, ctypes.byref(ms)) != 0:
            raise NNCError(100, _kern.nncb_last_error().decode())
        return ms.value

    def sync(self):
        _kern.nncb_sync(self.ctx)

    def launches(self) -> int:
        return int(_kern.nncb_launch_count(self.ctx))


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_host.nnc_comm_unique_id(buf))
    return buf.raw


def sync_stats(reset: bool = False) -> Dict[str, int]:
    """Device transfer counters (the reference's OffloadDevice::sync_stats)."""
    h, d, w = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(_host.nnc_device_sync_stats(1 if reset else 0, ctypes.byref(h), ctypes.byref(d), ctypes.byref(w)))
    return {"h2d_bytes": h.value, "d2h_bytes": d.value, "weight_bytes": w.value}


def init_comm(nranks: int, rank: int, uid: bytes):
    _check(_host.nnc_init_comm(nranks, rank, uid))


__all__ = ["load_native", "CompiledModel", "DeviceTimer", "NNCError", "group_document", "comm_unique_id",
           "init_comm", "PREC_TF32", "PREC_FP32", "PREC_BF16", "PREC_TF32X3", "HOST_LIB", "KERNEL_LIB"]
