"""Direct ctypes access to libnncb.so kernels (the thin C-ABI of include/nncb.h)
for kernel-level GPU tests."""
import ctypes

import numpy as np

import paper_2205_10357_b200 as P

K = P._kern
_P, _I, _I64, _D, _S = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_char_p


class GemmDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("kind", "precision", "epilogue", "tile")] + \
               [(n, ctypes.c_int64) for n in ("n", "ih", "iw", "ci", "co", "kh", "kw", "sh", "sw", "oh", "ow",
                                              "pad_top", "pad_left", "batch", "in_f", "out_f")] + \
               [("colstats", ctypes.c_void_p), ("eg_mask", ctypes.c_void_p), ("eg_res", ctypes.c_void_p),
                ("eg_x", ctypes.c_void_p), ("eg_stats", ctypes.c_void_p), ("eg_sums", ctypes.c_void_p),
                ("b_kmajor", ctypes.c_void_p), ("bn_mean", ctypes.c_void_p), ("bn_var", ctypes.c_void_p),
                ("bn_gamma", ctypes.c_void_p), ("bn_beta", ctypes.c_void_p), ("bn_eps", ctypes.c_double),
                ("residual", ctypes.c_void_p), ("sgd_w", ctypes.c_void_p), ("sgd_lr", ctypes.c_void_p),
                ("sgd_scale", ctypes.c_double), ("colstats_finalize", ctypes.c_void_p),
                ("colstats_eps", ctypes.c_double)]


class TransposeJob(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
                ("tile0", ctypes.c_int64)]


for name, res, args in [
    ("nncb_malloc", _I, [_P, ctypes.c_size_t, ctypes.POINTER(_P)]),
    ("nncb_free", _I, [_P, _P]),
    ("nncb_h2d", _I, [_P, _P, _P, ctypes.c_size_t]),
    ("nncb_d2h", _I, [_P, _P, _P, ctypes.c_size_t]),
    ("nncb_memset", _I, [_P, _P, _I, ctypes.c_size_t]),
    ("nncb_gemm", _I, [_P, ctypes.POINTER(GemmDesc), _P, _P, _P, _P]),
    ("nncb_gemm_last_path", _I, []),
    ("nncb_gemm_set_manual_a", _I, [_I]),
    ("nncb_gemm_force_tile", _I, [_I]),
    ("nncb_launch_count", ctypes.c_uint64, [_P]),
    ("nncb_transpose_batch", _I, [_P, _P, _I, ctypes.c_int64]),
]:
    fn = getattr(K, name)
    fn.restype, fn.argtypes = res, args


class EwInstr(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("dst", ctypes.c_int32), ("a", ctypes.c_int32), ("b", ctypes.c_int32),
                ("c", ctypes.c_int32), ("d", ctypes.c_int32), ("e", ctypes.c_int32), ("f", ctypes.c_int32),
                ("h", ctypes.c_int32), ("slot", ctypes.c_int32), ("imm", ctypes.c_double)]


class EwProgram(ctypes.Structure):
    _fields_ = [("n_instr", ctypes.c_int32), ("instr", ctypes.POINTER(EwInstr)), ("n_regs", ctypes.c_int32),
                ("n_slots", ctypes.c_int32)]


for name, res, args in [
    ("nncb_ew_compile", _I, [_P, ctypes.POINTER(EwProgram), ctypes.POINTER(_P)]),
    ("nncb_ew_launch", _I, [_P, _P, ctypes.POINTER(_P), ctypes.c_int64, ctypes.c_int64]),
    ("nncb_bn_grad_reduce", _I, [_P, _P, _P, _P, _P, _P, ctypes.c_int64, ctypes.c_int64]),
    ("nncb_sync", _I, [_P]),
    ("nncb_event_create", _I, [ctypes.POINTER(_P)]),
    ("nncb_event_record", _I, [_P, _P]),
    ("nncb_event_elapsed_ms", _I, [_P, _P, ctypes.POINTER(ctypes.c_float)]),
]:
    fn = getattr(K, name)
    fn.restype, fn.argtypes = res, args


def ew_run(instrs, n_regs, slots, n, channels):
    """Compile and launch a fused elementwise program; slots are Dev objects."""
    arr = (EwInstr * len(instrs))(*[EwInstr(**i) for i in instrs])
    prog = EwProgram(len(instrs), arr, n_regs, len(slots))
    kern = _P()
    rc = K.nncb_ew_compile(ctx(), ctypes.byref(prog), ctypes.byref(kern))
    assert rc == 0, K.nncb_last_error()
    ptrs = (_P * len(slots))(*[s.p for s in slots])
    rc = K.nncb_ew_launch(ctx(), kern, ptrs, n, channels)
    assert rc == 0, K.nncb_last_error()
    K.nncb_sync(ctx())


def ctx():
    c = P._host.nnc_device_ctx()
    assert c, P._host.nnc_last_error()
    return c


class Dev:
    def __init__(self, arr=None, nbytes=None):
        self.c = ctx()
        self.nbytes = arr.nbytes if arr is not None else nbytes
        self.p = _P()
        assert K.nncb_malloc(self.c, max(self.nbytes, 16), ctypes.byref(self.p)) == 0
        if arr is not None:
            a = np.ascontiguousarray(arr, dtype=np.float32)
            assert K.nncb_h2d(self.c, self.p, a.ctypes.data, a.nbytes) == 0
        else:
            K.nncb_memset(self.c, self.p, 0, self.nbytes)

    def get(self, shape):
        out = np.empty(shape, dtype=np.float32)
        assert K.nncb_d2h(self.c, out.ctypes.data, self.p, out.nbytes) == 0
        K.nncb_sync(self.c)
        return out

    def __del__(self):
        K.nncb_free(self.c, self.p)


def gemm(desc, a, b, bias, out):
    rc = K.nncb_gemm(ctx(), ctypes.byref(desc), a.p, b.p, bias.p if bias is not None else None, out.p)
    assert rc == 0, K.nncb_last_error().decode()
    assert K.nncb_sync(ctx()) == 0, K.nncb_last_error().decode()
