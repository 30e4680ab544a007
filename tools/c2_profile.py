import sys, os
sys.path.insert(0, "/root/repo")
import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
shape=(256,128,128,64)
x=W.uniform(shape,5,"x"); y=W.uniform(shape,6,"y")
m=P.CompiledModel(W.c2_chain(shape,'bn',batch_stats=True), precision=P.PREC_TF32)
m.run({"x":x,"y":y}, outputs=[])
for _ in range(2): prof=m.profile_run({"x":x,"y":y})
for p in prof: print(p['label'][:60], p['kind'], round(p['ms'],3), round(p['bytes']/1e9,2), round(p['bytes']/p['ms']/1e6 if p['ms'] else 0,1))
