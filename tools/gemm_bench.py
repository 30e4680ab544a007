"""Micro-benchmark of the tcgen05 GEMM (nncb_gemm, kind::tf32) on the ResNet-50
layer shapes at batch 256: per (layer, kind) device time from CUDA events over
repeated launches, useful TFLOP/s = 2*N*OH*OW*CO*KH*KW*CI / time.

    python tools/gemm_bench.py [--kinds fwd,dgrad,wgrad] [--reps 5] [--layers s0b,s2b]

Kernel tuning knobs are read from the environment by gemm_tc.cu (NNCB_TC_*)."""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2205_10357_b200 as P  # noqa: E402
from tests.nncb_ctypes import Dev, GemmDesc, K, ctx  # noqa: E402

LAYERS = [  # name, h(=w) in, ci, co, k, s   (ResNet-50, batch 256)
    ("stem", 224, 3, 64, 7, 2),
    ("s0b_a", 56, 256, 64, 1, 1), ("s0b_b", 56, 64, 64, 3, 1), ("s0b_c", 56, 64, 256, 1, 1),
    ("s1b0_b", 56, 128, 128, 3, 2), ("s1b_b", 28, 128, 128, 3, 1), ("s1b_c", 28, 128, 512, 1, 1),
    ("s1b_a", 28, 512, 128, 1, 1), ("s2b_b", 14, 256, 256, 3, 1), ("s2b_c", 14, 256, 1024, 1, 1),
    ("s3b_b", 7, 512, 512, 3, 1), ("s3b_c", 7, 512, 2048, 1, 1), ("s3b_a", 7, 2048, 512, 1, 1),
]


def geom(n, h, ci, co, k, s):
    oh = -(-h // s)
    pt = max((oh - 1) * s + k - h, 0) // 2
    return dict(n=n, ih=h, iw=h, ci=ci, co=co, kh=k, kw=k, sh=s, sw=s, oh=oh, ow=oh, pad_top=pt, pad_left=pt)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="fwd,dgrad,wgrad")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--layers", default="")
    ap.add_argument("--colstats", action="store_true", help="forward GEMMs also accumulate BN column statistics")
    ap.add_argument("--precision", type=int, default=0, help="0 tf32, 1 exact fp32, 2 bf16 operands")
    ap.add_argument("--dense", default="", help="dense shapes batch:in:out,... instead of conv layers")
    ap.add_argument("--eg", action="store_true", help="dgrad GEMMs run the ReLU-gradient + BN-sums epilogue")
    ap.add_argument("--bn", action="store_true", help="forward GEMMs run the inference BatchNorm + ReLU epilogue")
    ap.add_argument("--res", action="store_true", help="with --eg: add a residual gradient")
    ap.add_argument("--tile", default="auto", help="auto | 128 | 256 | p128 | p256 | w128 | t128 | h64 | th128 ... (p = CTA pair, w = wide staging, t = K-major weights, h = halo patches)")
    a = ap.parse_args()
    timer = P.DeviceTimer()
    if a.tile != "auto":
        t = a.tile
        code = (int(t.lstrip("pwthfr")) | (0x10000 if "p" in t else 0) | (0x20000 if "w" in t else 0) |
                (0x40000 if "t" in t else 0) | (0x80000 if "h" in t else 0) | (0x100000 if "f" in t else 0) |
                (0x200000 if "r" in t else 0))
        K.nncb_gemm_force_tile(code)
    total = {}
    for spec in [x for x in a.dense.split(",") if x]:
        bsz, fin, fout = (int(v) for v in spec.split(":"))
        flops = 2.0 * bsz * fin * fout
        X, Wt, Y = Dev(nbytes=bsz * fin * 4), Dev(nbytes=fin * fout * 4), Dev(nbytes=bsz * fout * 4)
        for kind in a.kinds.split(","):
            code, A, B, O = {"fwd": (0, X, Wt, Y), "dgrad": (1, Y, Wt, X), "wgrad": (2, X, Y, Wt)}[kind]
            d = GemmDesc(kind=code, precision=a.precision, batch=bsz, in_f=fin, out_f=fout)
            assert K.nncb_gemm(ctx(), ctypes.byref(d), A.p, B.p, None, O.p) == 0, K.nncb_last_error()
            timer.start()
            for _ in range(a.reps):
                K.nncb_gemm(ctx(), ctypes.byref(d), A.p, B.p, None, O.p)
            ms = timer.stop() / a.reps
            print(f"dense {spec} {kind:5s} {ms*1000:8.1f} us {flops/ms/1e9:7.1f} TF/s", flush=True)
    for name, h, ci, co, k, s in LAYERS:
        if a.dense:
            break
        if a.layers and not any(name.startswith(x) for x in a.layers.split(",")):
            continue
        g = geom(a.batch, h, ci, co, k, s)
        flops = 2.0 * a.batch * g["oh"] * g["ow"] * co * k * k * ci
        x = Dev(nbytes=a.batch * h * h * ci * 4)
        y = Dev(nbytes=a.batch * g["oh"] * g["ow"] * co * 4)
        w = Dev(nbytes=k * k * ci * co * 4)
        for kind in a.kinds.split(","):
            if kind == "dgrad" and ci % 32 and k > 1:
                continue   # the stem's input gradient is never needed (and has no tensor-core lowering)
            code, A, B, O = {"fwd": (3, x, w, y), "dgrad": (4, y, w, x), "wgrad": (5, x, y, w)}[kind]
            cs = Dev(nbytes=2 * co * 8) if (a.colstats and kind == "fwd") else None
            d = GemmDesc(kind=code, precision=a.precision, epilogue=4 if cs else 0, **g)
            if cs:
                d.colstats = cs.p
            if a.bn and kind == "fwd":
                bnp = [Dev(np.full(co, v, np.float32)) for v in (0.1, 1.0, 0.9, 0.05)]
                d.epilogue |= 32 | 2
                d.bn_mean, d.bn_var, d.bn_gamma, d.bn_beta = (t.p for t in bnp)
                d.bn_eps = 1e-5
            if a.eg and kind == "dgrad":
                eg = [Dev(nbytes=a.batch * h * h * ci * 4) for _ in range(3)] + [Dev(nbytes=2 * ci * 4), Dev(nbytes=2 * ci * 8)]
                d.epilogue = 8
                d.eg_mask, d.eg_x, d.eg_stats, d.eg_sums = eg[0].p, eg[1].p, eg[3].p, eg[4].p
                d.eg_res = eg[2].p if a.res else None
            rc = K.nncb_gemm(ctx(), ctypes.byref(d), A.p, B.p, None, O.p)   # warm-up
            assert rc == 0, K.nncb_last_error()
            timer.start()
            for _ in range(a.reps):
                K.nncb_gemm(ctx(), ctypes.byref(d), A.p, B.p, None, O.p)
            ms = timer.stop() / a.reps
            total[kind] = total.get(kind, 0) + ms
            print(f"{name:7s} {kind:5s} {ms*1000:8.1f} us {flops/ms/1e9:7.1f} TF/s", flush=True)
    print("totals (ms, one instance per layer shape):", {k: round(v, 3) for k, v in total.items()})


if __name__ == "__main__":
    main()
