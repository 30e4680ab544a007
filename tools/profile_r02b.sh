#!/usr/bin/env bash
# Round-2 evidence refresh after the elementwise load-ring changes: bench lines
# of every config, the C4 per-launch events, the reference arm, the ncu launch
# list, and `ncu --set full` of the relu-grad + reduction group and the C2
# statistics pass. Run on a GPU box from the repo root:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/profile_r02b.sh'
set -u
OUT=gpurun_out/prof
mkdir -p "$OUT"
python bench.py --steps 10 --warmup 3 --profile-json "$OUT/c4_per_launch_events.json" > "$OUT/bench_c4.json" 2> "$OUT/bench.log" || exit 1
tail -1 "$OUT/bench_c4.json" | cut -c1-200
for c in c1 c2 c3 c5; do
    python bench.py --config $c --no-cpu-baseline > "$OUT/bench_$c.json" 2>> "$OUT/bench.log" || exit 1
    tail -1 "$OUT/bench_$c.json" | cut -c1-160
done
python bench.py --impl reference > "$OUT/bench_ref.json" 2>> "$OUT/bench.log" || exit 1
tail -1 "$OUT/bench_ref.json" | cut -c1-160
SHORT="python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file "$OUT/c4_launches_ncu.csv" $SHORT > "$OUT/ncu_launches.log" 2>&1
EW="python tools/ew_bench.py --reps 2"
$EW > "$OUT/ew_plain.log" 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nnc_fused_ew -s 3 -c 1 \
    -o "$OUT/ew_relu_grad_reduce" -f $EW > "$OUT/ncu_ew.log" 2>&1
python tools/c2_profile.py > "$OUT/c2_plain.log" 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nnc_fused_ew -s 2 -c 1 \
    -o "$OUT/ew_c2_stats_pass" -f python tools/c2_profile.py > "$OUT/ncu_c2.log" 2>&1
echo done
