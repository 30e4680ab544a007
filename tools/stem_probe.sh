# stem conv (7x7/2, 3 -> 64 ch, batch 256): space-to-depth (default) vs im2col lowering
set -u
timeout 200 python tools/gemm_bench.py --layers stem --kinds fwd,wgrad --reps 10 2>&1 | grep -v totals
NNCB_TC_STEM=im2col timeout 200 python tools/gemm_bench.py --layers stem --kinds fwd,wgrad --reps 10 2>&1 | grep -v totals
