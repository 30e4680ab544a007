"""Regenerates paper_2205_10357_b200/csrc/kernels/tile_table.inc: runs the
BASELINE workloads (C1, C3/C4 ResNet-50-shaped, C5 MLP; C2 has no GEMMs), in the
tf32 and bf16 precisions, with
NNCB_TC_AUTOTUNE=fresh on a B200 so every GEMM shape they launch is measured
(the committed table is not consulted)
(candidates timed on a scratch output), then writes the chosen tile per shape.
The committed table makes the default (table) mode deterministic across
processes and boxes. Run under gpurun:  python tools/tune_tiles.py [out.inc]"""
import ctypes
import os
import sys

os.environ["NNCB_TC_AUTOTUNE"] = "fresh"   # live, without consulting the committed table
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_10357_b200 as P  # noqa: E402
from paper_2205_10357_b200 import workloads as W  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(P.__file__), "csrc", "kernels",
                                                               "tile_table.inc")
    P.load_native()
    cases = [("c1", W.c1_small_cnn(32, bn=True), {"x": W.uniform((32, 32, 32, 3), 1, "x")}, (32, 10)),
             ("c4", W.resnet50(256, bn=True), {"x": W.uniform((256, 224, 224, 3), 1, "x")}, (256, 1000)),
             ("c5", W.mlp(8192, 4096, 8), {"x": W.uniform((8192, 4096), 1, "x")}, (8192, 4096))]
    for name, doc, inputs, tshape in cases:
        for prec, pname in ((P.PREC_TF32, "tf32"), (P.PREC_BF16, "bf16")):
            if name == "c1" and pname == "bf16":
                continue
            m = P.CompiledModel(doc, precision=prec)
            t = W.uniform(tshape, 2, "t", 0.0, 1.0)
            m.trainer_prepare(inputs, t)          # first eager step: every training GEMM shape
            m.run(inputs)                         # inference (C3 for the ResNet-50-shaped graph)
            print(name, pname, "tuned", flush=True)
            del m
    k = P._kern
    k.nncb_gemm_tuning_export.restype = ctypes.c_int
    k.nncb_gemm_tuning_export.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    n = ctypes.c_size_t()
    k.nncb_gemm_tuning_export(None, 0, ctypes.byref(n))
    buf = ctypes.create_string_buffer(n.value)
    k.nncb_gemm_tuning_export(buf, n.value, ctypes.byref(n))
    lines = [ln for ln in buf.value.decode().splitlines() if ln.strip()]
    with open(out, "w") as f:
        f.write("// Per-shape tcgen05 GEMM tile choices, measured on a B200 by tools/tune_tiles.py\n"
                "// (key: gemm_tc tile key; choice: width | pair<<16 | wide<<17 | kmajor<<18 | halo<<19).\n")
        for ln in sorted(lines):
            key, choice = ln.rsplit(" ", 1)
            f.write('{"%s", %d},\n' % (key, int(choice)))
    print(f"{len(lines)} shapes -> {out}")


if __name__ == "__main__":
    main()
