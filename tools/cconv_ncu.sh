# ncu --set full of the s0 1x1 expansion conv (64 -> 256 ch, 56x56, batch 256)
# with and without the fused BatchNorm column-statistics epilogue
set -u
OUT=gpurun_out/prof; mkdir -p $OUT
G="python tools/gemm_bench.py --layers s0b_c --kinds fwd --reps 2"
$G > $OUT/cconv_plain.log 2>&1 || exit 1
$G --colstats > $OUT/cconv_cs.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -o $OUT/gemm_s0b_c_fwd $G > $OUT/ncu_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -o $OUT/gemm_s0b_c_fwd_cs $G --colstats > $OUT/ncu_c2.log 2>&1
echo done
