#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 backend (driver contract).

Default workload (BASELINE.json metric "fwd+bwd samples/sec (ResNet-50-shaped
graph)"): C4 = the ResNet-50-shaped graph with BatchNorm, one full training
step (forward, L1 loss, backward, SGD) at batch 256 per GPU, fp32 storage with
tcgen05 tf32 GEMMs, synthetic U(-1,1) inputs (activations are far larger than
the 126 MB L2, so no flush is needed between steps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4|c5] [--impl ours|reference]

Under torchrun (N > 1) every rank trains its own batch shard (weak scaling) and
gradients are all-reduced with NCCL inside the step's CUDA graph; rank 0 prints
one JSON line with the max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

CONFIGS = {
    "c1": dict(workload="C1 small CNN (conv-BN-ReLU-maxpool x2, dense, L1) train step", batch=32, kind="train"),
    "c2": dict(workload="C2 depth-16 BN/ReLU/Mul/Add chain on [256,128,128,64] fp32, train-mode BN forward",
               batch=256, kind="chain"),
    "c3": dict(workload="C3 ResNet-50-shaped (BN) inference", batch=256, kind="infer"),
    "c4": dict(workload="C4 ResNet-50-shaped (BN) training step fwd+L1+bwd+SGD", batch=256, kind="train"),
    "c5": dict(workload="C5 MLP 4096x8 (Dense+GELU+LayerNorm) training step", batch=8192, kind="train"),
}


def ncu_summary():
    """Newest profiles/r*/ncu_summary.json (written from this repo's ncu captures)."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*",
                                          "ncu_summary.json")))
    if not files:
        return {}
    with open(files[-1]) as f:
        return json.load(f)


TF32_PEAK_FILE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02", "tf32_peak.json")


def tf32_peak():
    """The tf32 dense peak measured with the driver's bf16 recipe (torch 8192^3,
    allow_tf32; tools/tf32_peak.py, committed under profiles/r02)."""
    try:
        with open(TF32_PEAK_FILE) as f:
            return json.load(f)
    except Exception:
        return None


def hbm_mix_note(achieved_gbs):
    """Read-heavy streams can run above the copy figure: the torch 2-read /
    1-write kernel measured on the same pool (tools/hbm_read_peak.py,
    profiles/r02/hbm_mix_peaks.json) as a second denominator."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02", "hbm_mix_peaks.json")
    try:
        mix = json.load(open(path))
    except (OSError, ValueError):
        return {}
    return {"peak_2r1w_gbs": mix["read2w1_gbs"], "frac_of_2r1w_peak": achieved_gbs / mix["read2w1_gbs"],
            "peak_2r1w_source": "profiles/r02/hbm_mix_peaks.json (torch.add(a, b, out=c), 1 Gi fp32, best of 10): "
                                "read-dominated traffic runs above the copy figure"}


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


class Clocks:
    """nvidia-smi sampling (clocks + throttle reasons) kept for the timed region.

    The sampler starts before the warm-up (nvidia-smi needs a few hundred ms to
    emit its first line); `mark_start` / `stop` bracket the timed region and
    only samples taken inside it are kept (or the nearest ones if the region is
    shorter than the sampling period)."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def mark_start(self):
        self.t0 = time.time()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.time(), parts))

    def stop(self):
        self.t1 = time.time()
        time.sleep(0.25)   # let the sample covering the region's end arrive
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        t0 = self.t0 if self.t0 is not None else self.t1
        inside = [p for t, p in self.samples if t0 <= t <= self.t1 + 0.1]
        if not inside and self.samples:   # region shorter than the period: nearest samples
            inside = [min(self.samples, key=lambda tp: abs(tp[0] - (t0 + self.t1) / 2))[1]]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm = []
        smax = None
        for s in inside:
            try:
                sm.append(float(s[0]))
                smax = float(s[1])
            except ValueError:
                continue
            for i, n in enumerate(names):
                if s[3 + i].lower() in ("active", "1", "yes"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(cfg: str, batch: int):
    from paper_2205_10357_b200 import workloads as W
    if cfg == "c1":
        doc = W.c1_small_cnn(batch, bn=True)
        inputs = {"x": W.uniform((batch, 32, 32, 3), 1, "x")}
        out_shape = (batch, 10)
    elif cfg == "c2":
        shape = (batch, 128, 128, 64)
        doc = W.c2_chain(shape, mode="bn", batch_stats=True)
        inputs = {"x": W.uniform(shape, 5, "x"), "y": W.uniform(shape, 6, "y")}
        out_shape = shape
    elif cfg in ("c3", "c4"):
        doc = W.resnet50(batch, bn=True)
        inputs = {"x": W.uniform((batch, 224, 224, 3), 1, "x")}
        out_shape = (batch, 1000)
    elif cfg == "c5":
        doc = W.mlp(batch, 4096, 8)
        inputs = {"x": W.uniform((batch, 4096), 1, "x")}
        out_shape = (batch, 4096)
    else:
        raise SystemExit(f"unknown config {cfg}")
    target = W.uniform(out_shape, 2, "target", 0.0, 1.0)
    return doc, inputs, target


def reference_doc(cfg: str, batch: int):
    """The reference's vocabulary has no BatchNorm / GELU / LayerNorm:
    its CPU arm runs the same graphs with those layers removed (labelled)."""
    from paper_2205_10357_b200 import workloads as W
    if cfg == "c1":
        return W.c1_small_cnn(batch, bn=False), {"x": W.uniform((batch, 32, 32, 3), 1, "x")}, (batch, 10)
    if cfg in ("c3", "c4"):
        return W.resnet50(batch, bn=False), {"x": W.uniform((batch, 224, 224, 3), 1, "x")}, (batch, 1000)
    if cfg == "c2":
        shape = (1, 128, 128, 64)
        return (W.c2_chain(shape, mode="ref"), {"x": W.uniform(shape, 5, "x"), "y": W.uniform(shape, 6, "y")},
                shape)
    if cfg == "c5":
        nodes = json.loads(W.mlp(batch, 4096, 8))
        nodes["nodes"] = [n for n in nodes["nodes"] if n["op"] == "dense"]
        for i, n in enumerate(nodes["nodes"]):
            n["inputs"] = ["x"] if i == 0 else [nodes["nodes"][i - 1]["name"]]
        nodes["outputs"] = [nodes["nodes"][-1]["name"]]
        return json.dumps(nodes), {"x": W.uniform((batch, 4096), 1, "x")}, (batch, 4096)
    raise SystemExit(cfg)


def _ref_worker(args):
    cfg, batch, seconds = args
    from oracle import reference as R
    from paper_2205_10357_b200 import workloads as W
    doc, inputs, out_shape = reference_doc(cfg, batch)
    m = R.RefModel(doc, 0)
    target = W.uniform(out_shape, 2, "target", 0.0, 1.0)
    n, t0 = 0, time.time()
    while True:
        if cfg == "c2" or cfg == "c3":
            m.run(inputs)
        else:
            m.train_step(inputs, target, 1e-4)
        n += 1
        if time.time() - t0 >= seconds:
            break
    return n, time.time() - t0


def cpu_reference(cfg: str, seconds: float, cores: int):
    """The reference CPU implementation (oracle/_ref, compiled from /root/reference
    sources) on the host cores: `cores` single-threaded replicas (the reference is
    single-threaded, plans are shareable), each stepping a reduced batch."""
    from multiprocessing import get_context
    batch = {"c1": 32, "c2": 1, "c3": 1, "c4": 1, "c5": 8}[cfg]
    with get_context("spawn").Pool(cores) as pool:
        res = pool.map(_ref_worker, [(cfg, batch, seconds)] * cores)
    steps = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    if cfg == "c2":
        elems = 128 * 128 * 64
        value = steps * elems * 12 / wall / 1e9
        unit = "GB/s"
    else:
        value = steps * batch / wall
        unit = "samples/s"
    sample = {"c1": "C1 without BatchNorm (reference vocabulary), batch 32 per replica",
              "c2": "C2 chain without BatchNorm, one [1,128,128,64] slice per step",
              "c3": "ResNet-50-shaped without BatchNorm, batch 1 inference per replica",
              "c4": "ResNet-50-shaped without BatchNorm, batch 1 train_step per replica",
              "c5": "MLP without GELU/LayerNorm (8 x Dense 4096), batch 8 per replica"}[cfg]
    return {"value": value, "unit": unit, "cores": cores, "kind": "reference",
            "sample": f"{sample}; {steps} steps in {wall:.1f} s on {cores} cores"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-json", default=None)
    ap.add_argument("--no-variants", action="store_true", help="skip the bf16 companion measurement")
    ap.add_argument("--precision", default="tf32", choices=["tf32", "bf16", "fp32", "tf32x3"],
                    help="GEMM precision: tf32 (default), bf16 operands for compute-bound contractions, exact fp32")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    cfg = CONFIGS[args.config]
    batch = args.batch or cfg["batch"]

    if args.impl == "reference":
        if rank != 0:
            return
        cores = min(os.cpu_count() or 1, 32)
        per_step = max(args.cpu_seconds / max(args.steps + args.warmup, 1), 2.0)
        cb = cpu_reference(args.config, per_step * max(args.steps, 1), cores)
        line = {"metric": cb["unit"] if args.config == "c2" else "fwd+bwd samples/sec (ResNet-50-shaped graph)"
                if args.config == "c4" else cb["unit"],
                "value": cb["value"], "unit": cb["unit"], "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "higher_is_better": True, "impl": "reference", "dtype": "f32",
                "data": "synthetic", "config": {"workload": cfg["workload"] + " (reference vocabulary)",
                                                "batch_per_replica": cb["sample"]},
                "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                                            "d2h_bytes_per_step": 0}, "vs_baseline": None}
        print(json.dumps(line), flush=True)
        return

    os.environ.setdefault("NNC_DEVICE", str(local))
    import paper_2205_10357_b200 as P
    from paper_2205_10357_b200 import workloads as W

    dist = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # the communicator shows in the logs
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("gloo", rank=rank, world_size=world)
        uid = [P.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        P.init_comm(world, rank, uid[0])

    doc, inputs, target = make_workload(args.config, batch)
    prec = {"tf32": P.PREC_TF32, "bf16": P.PREC_BF16, "fp32": P.PREC_FP32, "tf32x3": P.PREC_TF32X3}[args.precision]
    model = P.CompiledModel(doc, precision=prec)
    timer = P.DeviceTimer()
    lr = 1e-4
    clocks = Clocks(local)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        if not dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if cfg["kind"] in ("train",):
        model.trainer_prepare(inputs, target)
        step = lambda: model.trainer_step_device(lr)  # noqa: E731
        units = batch * world
        metric = "fwd+bwd samples/sec (ResNet-50-shaped graph)" if args.config == "c4" else "train samples/sec"
        unit = "samples/s"
    elif cfg["kind"] == "infer":
        model.run(inputs)
        step = lambda: model.run_device("inference")  # noqa: E731
        units = batch * world
        metric, unit = "inference samples/sec", "samples/s"
    else:  # chain: train-mode BN forward, reported as algorithmic HBM GB/s (SURVEY.md §8(d) C2 mode B)
        # the chain's BatchNorms use batch statistics in the inference-role plan
        # (no SaveSet for a backward); its bytes are the executed plan's own
        # algorithmic bytes (materialize-at-barrier: every launch's reads and
        # writes, counted once), measured per launch below
        model.run(inputs, role="inference", outputs=[])
        step = lambda: model.run_device("inference")  # noqa: E731
        prof_c2 = model.profile_run(inputs, "inference")
        plan_bytes = sum(p["bytes"] for p in prof_c2)
        elems = int(np.prod(inputs["x"].shape))
        units = plan_bytes * world / 1e9   # GB per pass
        metric, unit = "fused-group HBM GB/s (C2 chain, train-mode BN)", "GB/s"

    clocks.start()   # sampler warms up during the warm-up steps
    for _ in range(args.warmup):
        step()
    timer.sync()
    barrier()
    clocks.mark_start()
    l0 = timer.launches()
    timer.start()
    for _ in range(args.steps):
        step()
    ms = timer.stop()
    clk = clocks.stop()
    launches = timer.launches() - l0
    if cfg["kind"] == "train":   # graph replays are not counted by the host-side counter
        launches = max(launches, model.launches_per_step() * args.steps)
    else:
        # inference / chain runs replay a CUDA graph: count one eager run's
        # kernel launches (profile_run enqueues every launch of the plan)
        la = timer.launches()
        model.profile_run(inputs, "inference")
        launches = max(launches, (timer.launches() - la) * args.steps)
    ms = max_over_ranks(ms)
    ms_per_step = ms / args.steps
    value = units / (ms_per_step / 1000.0)

    # ---- end to end through the public API (host buffers every step) ----
    e2e = None
    if cfg["kind"] in ("infer", "chain"):
        role = "inference"   # C2 included: its forward-only plan (batch statistics, no SaveSet)
        h2d = sum(v.nbytes for v in inputs.values())
        final = [v["name"] for v in model.describe[role]["values"] if v["category"] == "output"]
        # the public pipelined loop: every run uploads its inputs from host memory
        # (the next run's upload overlaps this run) and downloads its outputs
        out = model.run_many([inputs] * 2, role=role, outputs=final)[-1]   # untimed warm-up
        d2h = sum(v.nbytes for v in out.values())
        timer.sync()
        barrier()
        t0 = time.perf_counter()
        n_e2e = max(3, args.steps)
        outs = model.run_many([inputs] * n_e2e, role=role, outputs=final)
        e_ms = max_over_ranks((time.perf_counter() - t0) * 1000 / n_e2e)
        assert len(outs) == n_e2e
        e2e = {"value": units / (e_ms / 1000.0), "unit": unit, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e_ms}
    if cfg["kind"] == "train":
        # the public pipelined loop: every step uploads its inputs + target from
        # host memory (the next step's upload overlaps this step's compute) and
        # reads its loss back
        h2d = sum(v.nbytes for v in inputs.values()) + target.nbytes
        n_e2e = max(3, args.steps)   # the first upload (not overlapped) amortised over as many steps as the device timing
        model.train_steps([(inputs, target)] * 2, lr)   # untimed warm-up of the public path
        timer.sync()
        barrier()
        t0 = time.perf_counter()
        timer.start()
        losses = model.train_steps([(inputs, target)] * n_e2e, lr)
        e_ms = timer.stop()
        wall = (time.perf_counter() - t0) * 1000
        assert len(losses) == n_e2e
        e_ms = max_over_ranks(max(e_ms, wall) / n_e2e)
        e2e = {"value": units / (e_ms / 1000.0), "unit": unit, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8,
               "ms_per_step": e_ms}

    # ---- roofline of the dominant kernel (per-launch CUDA events) ----
    roof, top, fused_roof = None, None, None
    if rank == 0:
        if cfg["kind"] == "train":
            prof = model.profile_step(0.0)
        elif cfg["kind"] == "infer":
            prof = model.profile_run(inputs, "inference")
        else:
            prof = prof_c2
        if args.profile_json:
            with open(args.profile_json, "w") as f:
                json.dump(prof, f, indent=1)
        # dominant kernel = the kernel FUNCTION with the largest share of the step
        # (all tcgen05 GEMM launches are one kernel; all generated fused groups
        # are "ew"); achieved = its algorithmic flops (or bytes) / its device time
        fam = {}
        for p in prof:
            k = p["kind"].split(":")[0]
            a = fam.setdefault(k, {"ms": 0.0, "bytes": 0.0, "flops": 0.0, "n": 0})
            a["ms"] += p["ms"]
            a["bytes"] += p["bytes"]
            a["flops"] += p["flops"]
            a["n"] += 1
        total = sum(a["ms"] for a in fam.values())
        pk, src = peaks()

        t32 = tf32_peak()

        def roofline(k, a):
            if a["flops"] > 0:
                ach = a["flops"] / (a["ms"] / 1000) / 1e12
                peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
                r = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                     "traffic": None, "kernel": k, "launches_per_step": a["n"],
                     "share_of_step": a["ms"] / total,
                     "peak_source": f"{src} bf16 dense sustained (tf32 runs at half the bf16 rate)"}
                if t32:
                    # the family computes in tf32: its own measured ceiling, and the
                    # per-launch roofline time (each GEMM bounded by max(flops / tf32
                    # peak, algorithmic bytes / HBM) -- many are 1x1 convs that are
                    # HBM-bound) over the measured time
                    tp = t32["tf32_tflops_sustained"]
                    ideal = sum(max(p["flops"] / (tp * 1e12), p["bytes"] / (pk["hbm_gbs"] * 1e9)) for p in prof
                                if p["kind"].split(":")[0] == k) * 1e3
                    r.update({"tf32_peak": tp, "frac_of_tf32_peak": ach / tp,
                              "tf32_peak_source": "profiles/r02/tf32_peak.json (torch fp32 matmul allow_tf32 8192^3, "
                                                  "back to back 4 s, the MEASURED_PEAKS recipe)",
                              "roofline_time_frac": ideal / a["ms"],
                              "roofline_time_note": "sum over launches of max(flops/tf32 peak, bytes/HBM peak) "
                                                    "divided by the family's measured time"})
                return r
            ach = a["bytes"] / (a["ms"] / 1000) / 1e9
            return {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / pk["hbm_gbs"], "traffic": None, "kernel": k, "launches_per_step": a["n"],
                    "share_of_step": a["ms"] / total, "peak_source": f"{src} HBM copy", **hbm_mix_note(ach)}

        top_k = max(fam, key=lambda k: fam[k]["ms"])
        roof = roofline(top_k, fam[top_k])
        if "ew" in fam:
            fused_roof = roofline("ew (generated fused groups)", fam["ew"])
        # DRAM traffic per launch from the committed `ncu --set full` capture of
        # a representative launch of each family, beside its algorithmic bytes
        ew_key = "ew_c2" if args.config == "c2" else "ew"   # the C2 statistics pass capture
        for r, fk in ((roof, ew_key if top_k == "ew" else top_k), (fused_roof, ew_key)):
            summ = ncu_summary().get(fk) if r else None
            if summ:
                r["traffic"] = summ["dram_read_bytes"] + summ["dram_write_bytes"]
                r["traffic_launch"] = {"launch": summ["launch"], "algorithmic_bytes": summ["algorithmic_bytes"],
                                       "source": summ["report"]}
        by_kind = {}
        for p in prof:
            k = p["kind"].split(":")[0]
            d = by_kind.setdefault(k, {"ms": 0.0, "bytes": 0.0, "flops": 0.0})
            d["ms"] += p["ms"]
            d["bytes"] += p["bytes"]
            d["flops"] += p["flops"]
        top = {k: {"ms": round(v["ms"], 3),
                   "GB/s": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1),
                   "TFLOP/s": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 1)} for k, v in by_kind.items()}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_reference(args.config, args.cpu_seconds, min(os.cpu_count() or 1, 32))
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "error": str(exc)[:200]}
    # the same workload in the other tensor-core modes, same timing rules, on
    # rank 0 of a single-GPU run, reported beside the headline: bf16 operand
    # copies for the compute-bound forward / input-gradient GEMMs
    # (NNCB_PREC_BF16), and the split-operand 3xTF32 route (NNCB_PREC_TF32X3)
    variant = None
    if (rank == 0 and world == 1 and args.precision == "tf32" and cfg["kind"] in ("train", "infer")
            and not args.no_variants):
        del model
        variant = {}
        for vname, vprec in (("bf16", P.PREC_BF16), ("tf32x3", P.PREC_TF32X3)):
            vm = P.CompiledModel(doc, precision=vprec)
            if cfg["kind"] == "train":
                vm.trainer_prepare(inputs, target)
                vstep = lambda: vm.trainer_step_device(lr)  # noqa: E731
            else:
                vm.run(inputs)
                vstep = lambda: vm.run_device("inference")  # noqa: E731
            for _ in range(args.warmup):
                vstep()
            timer.sync()
            timer.start()
            for _ in range(args.steps):
                vstep()
            v_ms = timer.stop() / args.steps
            variant[vname] = {"value": units / (v_ms / 1000.0), "unit": unit, "ms_per_step": v_ms}
            del vm
        variant["bf16"].update({
            "dtype": "f32 storage; tcgen05 kind::f16 on bf16 operand copies for the compute-bound forward / "
                     "input-gradient GEMMs (arithmetic intensity >= 128), tf32 for the rest; fp32 accumulate",
            "parity": "tests/test_gpu_baseline_parity.py (bf16 rows): launch by launch within 2e-2 of the float64 "
                      "truth"})
        variant["tf32x3"].update({
            "dtype": "f32; every GEMM on tcgen05 kind::tf32 over split operands (hi + lo, K concatenated 3x): "
                     "1e-5-class GEMM error; exact elementwise ops",
            "parity": "tests/test_gpu_tf32x3.py (kernels vs float64) and tests/test_gpu_baseline_parity.py "
                      "(tf32x3 row: the C4 step launch by launch against the float64 truth)"})
    mode_a = None
    if cfg["kind"] == "chain" and rank == 0:
        # SURVEY.md §8(d) C2 mode A: inference BatchNorm (per-channel affine),
        # the whole chain one fused group: read x, y, write out = 12 B/element
        model = P.CompiledModel(W.c2_chain(tuple(inputs["x"].shape), mode="bn"), precision=P.PREC_TF32)
        model.run(inputs, role="inference", outputs=[])
        for _ in range(3):
            model.run_device("inference")
        timer.sync()
        timer.start()
        for _ in range(args.steps):
            model.run_device("inference")
        a_ms = timer.stop() / args.steps
        elems = int(np.prod(inputs["x"].shape))
        pk, src = peaks()
        gbs = 12.0 * elems / (a_ms / 1000.0) / 1e9
        mode_a = {"metric": "fused-group HBM GB/s (C2 chain, inference BN)", "value": gbs, "unit": "GB/s",
                  "ms_per_pass": a_ms, "bytes_per_element": 12, "frac_of_hbm_peak": gbs / pk["hbm_gbs"],
                  "peak_source": f"{src} HBM copy", **hbm_mix_note(gbs)}
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": {"tf32": "f32 (tcgen05 kind::tf32 GEMMs, fp32 accumulate)",
                                       "bf16": "f32 storage; tcgen05 kind::f16 on bf16 operand copies for the "
                                               "compute-bound forward / input-gradient GEMMs, tf32 for the rest; "
                                               "fp32 accumulate",
                                       "fp32": "f32 (exact-order fp32 GEMMs)",
                                       "tf32x3": "f32 (split-operand 3xTF32 tcgen05 GEMMs, fp32 accumulate)"}[
                                           args.precision],
        "data": "synthetic",
        "config": {"workload": cfg["workload"], "global_batch": batch * world, "batch_per_gpu": batch,
                   "parallelism": f"dp{world}", "l2": "activations >> 126 MB L2; no flush needed"},
        "clocks": clk, "e2e": e2e, "gpu_launches": launches, "roofline": roof, "fused_group_roofline": fused_roof,
        "cpu_baseline": cpu,
        "by_kernel_kind": top,
    }
    if variant:
        line["precision_variants"] = variant
    if mode_a:
        line["mode_a"] = mode_a
        line["config"]["note"] = ("value = mode B: train-mode BN forward (batch statistics, 4 barriers) as a "
                                  "forward-only plan; GB = the executed plan's algorithmic bytes (%.1f B/element: "
                                  "statistics passes recompute the chain from x, y instead of storing each "
                                  "barrier's input -- SURVEY 8(d)'s 40; NNC_NO_STATS_RECOMPUTE=1 gives the "
                                  "materializing plan, 64); mode_a = inference-BN chain, one fused pass "
                                  "(12 B/element)" % (plan_bytes / elems))
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
