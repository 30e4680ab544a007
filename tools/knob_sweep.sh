set -u
run() { echo -n "$1: "; env $1 timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],1),round(d['ms_per_step'],3),d['clocks']['sm_mhz'])"; }
run NONE=1
run NNCB_EW_RED_BLOCKS=2
run NNCB_EW_RED_BLOCKS=8
run NNCB_EW_MINBLOCKS=2
run NNCB_EW_MINBLOCKS=4
run NNC_BN_STATS_FUSE_MIN_K=128
run NNCB_TC_STGBUF=1
run NONE=2
