"""Reads the NNCB_TC_TRACE probe dump of tc_gemm_kernel launches (per CTA and
local tile: 0 MMA tile start (after tmem_empty), 1 MMA commit issued, 2
epilogue warp 2 saw tmem_full, 3 its TMEM release, 4 warp 2 tile done, 5 warp
9 tile done, 6 producer tile start; %globaltimer ns) and prints the per-tile
phase durations averaged over CTAs."""
import sys

import numpy as np

data = open(sys.argv[1], "rb").read()
off = 0
while off < len(data):
    hdr = np.frombuffer(data, dtype=np.int64, count=6, offset=off)
    off += 48
    grid, tiles, bn, stages, stg_bufs, per_sm = (int(v) for v in hdr)
    ev = np.frombuffer(data, dtype=np.uint64, count=grid * 64 * 8, offset=off).reshape(grid, 64, 8).astype(np.float64)
    off += grid * 64 * 8 * 8
    per = min(64, -(-tiles // grid))
    e = ev[:, :per, :]
    t0 = e[:, 0, 6].min()
    e = (e - t0) / 1000.0   # us
    print(f"launch grid={grid} tiles={tiles} bn={bn} stages={stages} stg_bufs={stg_bufs} per_sm={per_sm} tiles/cta={per}")
    mma_issue = e[:, :, 1] - e[:, :, 0]
    mma_wait = e[:, 1:, 0] - e[:, :-1, 1]
    to_epi = e[:, :, 2] - e[:, :, 1]
    epi = e[:, :, 4] - e[:, :, 2]
    hold = e[:, :, 3] - e[:, :, 2]
    epi_gap = e[:, 1:, 2] - e[:, :-1, 4]
    total = e[:, per - 1, 4].max()
    print(f"  total {total:.1f} us; per tile: MMA issue {np.median(mma_issue):.2f}, MMA waits for TMEM "
          f"{np.median(mma_wait):.2f}, commit->epilogue {np.median(to_epi):.2f}, epilogue {np.median(epi):.2f} "
          f"(TMEM held {np.median(hold):.2f}), epilogue idle between tiles {np.median(epi_gap):.2f}")
    c = int(np.argmax(e[:, per - 1, 4]))
    print("  CTA", c, "tile timeline (us): [mma0, mma1, epi2, rel3, end4, end9, prod6]")
    for l in range(min(per, 6)):
        print("   ", l, np.round(e[c, l], 2))
