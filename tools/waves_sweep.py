#!/usr/bin/env python
"""Sweep of the auto chunk length's wave count (option "waves": the chunks
fill this many waves of co-resident filter-finish threads) for PRTS at
T = 2^log2t on the tracking model, device-resident, CUDA events on the
library's stream.  usage: python tools/waves_sweep.py [--log2t 24]
[--waves 2,3,4,5,6,8] [--dtypes f64,f32] [--reps 10]"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import numpy as np
    import torch

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_matrices, simulate_cv

    ap = argparse.ArgumentParser()
    ap.add_argument("--log2t", type=int, default=24)
    ap.add_argument("--waves", default="2,3,4,5,6,8")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    T = 1 << args.log2t
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    F, Q, H, R, m0, P0 = cv_matrices()
    ys_np = simulate_cv(T, seed=1)
    for dts in args.dtypes.split(","):
        tdt = torch.float64 if dts == "f64" else torch.float32

        def field(a):
            t = torch.as_tensor(a, dtype=tdt, device=dev)
            return t.expand(T, *t.shape).contiguous()

        m = psk.Lgssm(f=field(F), u=field(np.zeros(4)), q=field(Q), h=field(H),
                      d=field(np.zeros(2)), r=field(R),
                      prior_mean=torch.as_tensor(m0, dtype=tdt, device=dev),
                      prior_cov=torch.as_tensor(P0, dtype=tdt, device=dev), t=T)
        ys = torch.as_tensor(ys_np, dtype=tdt, device=dev)
        out = psk.GaussianStats(torch.empty((T, 4), dtype=tdt, device=dev),
                                torch.empty((T, 4, 4), dtype=tdt, device=dev))
        spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback)
        for w in [int(x) for x in args.waves.split(",")]:
            be = psk.CudaBackend(0, stream=stream)
            if w > 0:  # 0: the library default
                be.set_option("waves", w)
            with torch.cuda.stream(stream):
                for _ in range(3):
                    psk.prts_run(m, ys, spec, be, out=out)
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.reps):
                    psk.prts_run(m, ys, spec, be, out=out)
                e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            print(json.dumps({"dtype": dts, "log2t": args.log2t, "waves": w, "ms": round(ms, 4),
                              "steps_per_s": T / (ms * 1e-3)}), flush=True)
        del m, ys, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
