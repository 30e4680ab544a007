"""Writes profiles/<round>/ncu_summary.json (+ raw CSV exports) from the ncu
reports tools/profile_round.sh leaves in gpurun_out/prof. Run here (ncu -i)."""
import csv, json, os, subprocess, sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(root, "gpurun_out", "prof")
dst = os.path.join(root, "profiles", rnd)
os.makedirs(dst, exist_ok=True)


def raw(name):
    out = os.path.join(dst, f"{name}_raw.csv")
    with open(out, "w") as f:
        subprocess.run(["ncu", "-i", os.path.join(src, f"{name}.ncu-rep"), "--page", "raw", "--csv"], stdout=f,
                       stderr=subprocess.DEVNULL, check=True)
    rows = list(csv.reader(open(out)))
    return {k: (v, u) for k, u, v in zip(rows[0], rows[1], rows[2])}


def num(d, k, scale=1.0):
    v, u = d[k]
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u.strip(), 1.0)
    return float(v.replace(",", "")) * (mult if scale == 1.0 else scale)


g, e, e2 = raw("gemm_s2b_b_fwd"), raw("ew_relu_grad_reduce"), raw("ew_c2_stats_pass")
summ = {
    "gemm": {"kernel": g["Kernel Name"][0].strip(),
             "launch": "conv fwd 3x3 s1, 256->256 ch, 14x14, batch 256 (ResNet-50 stage-2 block b), tools/gemm_bench.py",
             "duration_us": float(g["gpu__time_duration.sum"][0]),
             "dram_read_bytes": num(g, "dram__bytes_read.sum"), "dram_write_bytes": num(g, "dram__bytes_write.sum"),
             "algorithmic_bytes": 256 * 14 * 14 * 256 * 4 * 2 + 3 * 3 * 256 * 256 * 4,
             "flops": 2.0 * 256 * 14 * 14 * 256 * 9 * 256,
             "tensor_pipe_active_pct": float(g["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]),
             "l2_to_smem_bytes": num(g, "l1tex__m_xbar2l1tex_read_bytes.sum"),
             "registers": float(g["launch__registers_per_thread"][0]),
             "report": f"profiles/{rnd}/gemm_s2b_b_fwd_raw.csv"},
    "ew": {"kernel": "nnc_fused_ew (relu-grad group + fused REDUCE_BN_GRAD)",
           "launch": "200704 x 128 (ResNet-50 stage-1 block b backward), tools/ew_bench.py",
           "duration_us": float(e["gpu__time_duration.sum"][0]),
           "dram_read_bytes": num(e, "dram__bytes_read.sum"), "dram_write_bytes": num(e, "dram__bytes_write.sum"),
           "algorithmic_bytes": 200704 * 128 * 4 * 4,
           "dram_throughput_pct": float(e["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
           "registers": float(e["launch__registers_per_thread"][0]),
           "report": f"profiles/{rnd}/ew_relu_grad_reduce_raw.csv"},
    "ew_c2": {"kernel": "nnc_fused_ew (C2 recomputed-statistics pass, REDUCE_STATS)",
              "launch": "C2 chain statistics pass over x, y [256,128,128,64] (reads 2 x 1.07 GB, stores nothing), "
                        "tools/c2_profile.py",
              "duration_us": float(e2["gpu__time_duration.sum"][0]),
              "dram_read_bytes": num(e2, "dram__bytes_read.sum"), "dram_write_bytes": num(e2, "dram__bytes_write.sum"),
              "algorithmic_bytes": 2 * 256 * 128 * 128 * 64 * 4,
              "dram_throughput_pct": float(e2["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
              "registers": float(e2["launch__registers_per_thread"][0]),
              "report": f"profiles/{rnd}/ew_c2_stats_pass_raw.csv"},
    "note": ("ncu --set full --clock-control none (serialised, cold per-kernel caches): compare shares and traffic, "
             "not absolute times. Writes still resident in the 126 MB L2 at kernel end are not counted in "
             "dram_write_bytes."),
}
json.dump(summ, open(os.path.join(dst, "ncu_summary.json"), "w"), indent=1)
print(json.dumps(summ, indent=1))
