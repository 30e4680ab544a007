set -u
OUT=gpurun_out/prof2
mkdir -p $OUT
GEMM="python tools/gemm_bench.py --layers s2b_b --kinds fwd --reps 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o "$OUT/gemm_s2b_b_fwd" $GEMM > "$OUT/ncu_gemm.log" 2>&1
GEMM16="python tools/gemm_bench.py --layers s2b_b --kinds fwd --reps 2 --precision 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o "$OUT/gemm_s2b_b_fwd_bf16" $GEMM16 > "$OUT/ncu_gemm16.log" 2>&1
GEMMD="python tools/gemm_bench.py --dense 8192:4096:4096 --kinds fwd --reps 2 --precision 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o "$OUT/gemm_dense4096_fwd_bf16" $GEMMD > "$OUT/ncu_gemmd.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nnc_fused_ew -s 2 -c 1 -o "$OUT/ew_c2_stats_pass" python tools/c2_profile.py > "$OUT/ncu_c2.log" 2>&1
SHORT="python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file "$OUT/c4_launches_ncu.csv" $SHORT > "$OUT/ncu_launches.log" 2>&1
ls -la $OUT
