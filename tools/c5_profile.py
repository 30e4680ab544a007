"""Per-launch profile of one C5 training step (MLP 4096 x 8, batch 8192):
families and the slowest launches."""
import sys
from collections import defaultdict
sys.path.insert(0, ".")
import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
prec = P.PREC_BF16 if "bf16" in sys.argv else P.PREC_TF32
m = P.CompiledModel(W.mlp(8192, 4096, 8), precision=prec)
x = {"x": W.uniform((8192, 4096), 1, "x")}
t = W.uniform((8192, 4096), 2, "t", 0.0, 1.0)
m.trainer_prepare(x, t)
prof = m.profile_step(0.0)
fam = defaultdict(lambda: [0.0, 0.0, 0.0, 0])
for p in prof:
    f = fam[p["kind"]]
    f[0] += p["ms"]; f[1] += p["bytes"]; f[2] += p["flops"]; f[3] += 1
print("total ms", round(sum(p["ms"] for p in prof), 3))
for k, (ms, b, fl, n) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} {ms:7.3f} ms  n={n:3d}  {b / ms / 1e6 if ms else 0:8.1f} GB/s  {fl / ms / 1e9 if ms else 0:7.1f} TF/s")
for p in sorted(prof, key=lambda p: -p["ms"])[:12]:
    print(p["label"][:50], p["kind"], round(p["ms"], 3), round(p["bytes"] / p["ms"] / 1e6), round(p["flops"] / p["ms"] / 1e9))
