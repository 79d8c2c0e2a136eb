"""Summarise a PSK_DLB_TRACE file: per-phase durations of the decoupled
look-back scan (fold, tile scan, look-back, apply) over all tiles."""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()  # usage: dlb_trace.py <PSK_DLB_TRACE file>
off = 0
while off < len(raw):
    nt, per, ks, n = np.frombuffer(raw, dtype=np.int64, count=4, offset=off)
    off += 32
    st = np.frombuffer(raw, dtype=np.uint64, count=int(nt) * 8, offset=off).reshape(-1, 8).astype(np.float64)
    off += int(nt) * 64
    t0 = st[:, 0].min()
    s = st - t0
    print(f"scan n={n} tiles={nt} per={per} elem={ks}: total {(st[:,5].max()-t0)/1e3:.1f} us")
    names = ["fold", "tile_scan", "publish+lookback", "publish P", "apply"]
    for i, nm in enumerate(names):
        d = (st[:, i + 1] - st[:, i]) / 1e3
        if i == 2:
            d = (st[:, 3] - st[:, 2]) / 1e3
        print(f"  {nm:18s} mean {np.mean(d[1:]):8.1f} us  max {np.max(d[1:]):8.1f} us")
    print(f"  start spread {(st[:,0].max()-t0)/1e3:.1f} us, last end {(st[:,5].max()-t0)/1e3:.1f} us")
