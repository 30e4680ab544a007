import sys; sys.path.insert(0,'.')
import numpy as np, paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W
doc=W.resnet50(2,bn=True); x=W.uniform((2,224,224,3),1,"x"); t=W.uniform((2,1000),2,"t",4.0,6.0)
m=P.CompiledModel(doc,precision=P.PREC_TF32); m.debug_keep_values(True); m.gradients({"x":x},t)
for v in m.describe["train_fwd"]["values"]:
    try: m.step_value(v["name"])
    except P.NNCError as e:
        if "never written" in str(e): print(v["name"], v["category"], v["storage"])
for role in ("train_bwd",):
    for v in m.describe[role]["values"]:
        try: m.step_value(v["name"])
        except P.NNCError as e:
            if "never written" in str(e): print(role, v["name"], v["category"], v["storage"])
