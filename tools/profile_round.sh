#!/usr/bin/env bash
# Round evidence for profiles/: the bench line, per-launch CUDA-event times,
# the ncu launch list of the same command, and one `ncu --set full` capture of
# the top GEMM and fused-EW kernels. Run on a GPU box from the repo root:
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/profile_round.sh'
# ncu steps run only after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/prof
mkdir -p "$OUT"
CMD="python bench.py --steps 10 --warmup 3"
$CMD --profile-json "$OUT/c4_per_launch_events.json" > "$OUT/bench_c4.json" 2> "$OUT/bench.log" || exit 1
tail -1 "$OUT/bench_c4.json"
SHORT="python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline"
$SHORT > "$OUT/plain.log" 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file "$OUT/c4_launches_ncu.csv" $SHORT > "$OUT/ncu_launches.log" 2>&1
# representative 3x3 convolution (s2 block, batch 256) and one fused group
GEMM="python tools/gemm_bench.py --layers s2b_b --kinds fwd --reps 2"
$GEMM > "$OUT/gemm_plain.log" 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 \
    -o "$OUT/gemm_s2b_b_fwd" $GEMM > "$OUT/ncu_gemm.log" 2>&1
# the same 3x3 convolution on the bf16 route (tcgen05 kind::f16)
GEMM16="python tools/gemm_bench.py --layers s2b_b --kinds fwd --reps 2 --precision 2"
$GEMM16 > "$OUT/gemm16_plain.log" 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 \
    -o "$OUT/gemm_s2b_b_fwd_bf16" $GEMM16 > "$OUT/ncu_gemm16.log" 2>&1
EW="python tools/ew_bench.py --reps 2"
$EW > "$OUT/ew_plain.log" 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nnc_fused_ew -s 3 -c 1 \
    -o "$OUT/ew_relu_grad_reduce" $EW > "$OUT/ncu_ew.log" 2>&1
echo done
