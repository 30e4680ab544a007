# 1x1 expansion convs (the BN-statistics "c" layers): colstats cost and tile choices
set -u
L=s0b_c,s1b_c,s2b_c,s3b_c
for t in auto 128 256 w128 p256; do
  echo "== tile $t plain"; timeout 120 python tools/gemm_bench.py --layers $L --kinds fwd --reps 10 --tile $t 2>&1 | grep -v totals
  echo "== tile $t colstats"; timeout 120 python tools/gemm_bench.py --layers $L --kinds fwd --reps 10 --tile $t --colstats 2>&1 | grep -v totals
done
