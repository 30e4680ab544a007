"""Per-launch CUDA-event profile of one C3 inference pass (ResNet-50-shaped,
batch 256): prints the GEMM launches with their times and algorithmic GB/s."""
import sys
sys.path.insert(0, ".")
import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
prec = P.PREC_BF16 if "bf16" in sys.argv else P.PREC_TF32
m = P.CompiledModel(W.resnet50(256, bn=True), precision=prec)
x = {"x": W.uniform((256, 224, 224, 3), 1, "x")}
m.run(x)
prof = m.profile_run(x)
tot = sum(p["ms"] for p in prof)
print("total ms", round(tot, 3), "launches", len(prof))
for p in prof:
    if "-v" in sys.argv or p["label"] in ("stem", "s0b1_a", "s0b1_b", "s0b1_c", "s2b1_b", "s2b1_c"):
        print(p["label"], p["kind"], round(p["ms"], 3), round(p["bytes"] / p["ms"] / 1e6))
