"""Break the end-to-end train_step (host buffers) into feed / step pieces."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2205_10357_b200 as P

doc, inputs, target = bench.make_workload("c4", 256)
m = P.CompiledModel(doc, precision=P.PREC_TF32)
m.train_step(inputs, target, 1e-4)
m.train_step(inputs, target, 1e-4)
for rep in range(3):
    t0 = time.perf_counter()
    for k, v in inputs.items():
        m.feed(k, v)
    t1 = time.perf_counter()
    t = np.ascontiguousarray(target, dtype=np.float32)
    import ctypes
    loss = ctypes.c_double()
    P._check(P._host.nnc_model_train_step(m._h, P._fptr(t), t.size, 1e-4, ctypes.byref(loss)))
    t2 = time.perf_counter()
    print(f"feed {1e3*(t1-t0):.2f} ms  train_step {1e3*(t2-t1):.2f} ms")
m.trainer_prepare(inputs, target)
for rep in range(3):
    t0 = time.perf_counter(); m.trainer_step_device(1e-4); m.trainer_loss(); t1 = time.perf_counter()
    print(f"device step {1e3*(t1-t0):.2f} ms")
