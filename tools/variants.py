#!/usr/bin/env python
"""BASELINE configs[1]: PKF / PRTS / PTFS time-steps/s per scan variant, T sweep,
FP32 and FP64, on one B200 (device-resident inputs, CUDA events on the
library's stream).  Prints one JSON line per (method, alg, dtype, T).

usage: python tools/variants.py [--log2t 10,14,18,20,22] [--dtypes f64,f32]
                                [--algs 1,2,3,4,5,6] [--methods prts] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_matrices, simulate_cv

    ap = argparse.ArgumentParser()
    ap.add_argument("--log2t", default="10,14,18,20,22")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--algs", default="1,2,3,4,5,6")
    ap.add_argument("--methods", default="prts")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--chunk", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    be = psk.CudaBackend(0, mode="fast", chunk=args.chunk, stream=stream)
    F, Q, H, R, m0, P0 = cv_matrices()
    for lt in [int(x) for x in args.log2t.split(",")]:
        T = 1 << lt
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
            for meth in args.methods.split(","):
                fn = getattr(psk, meth + "_run")
                for alg in [int(a) for a in args.algs.split(",")]:
                    spec = psk.ScanSpec(psk.ScanAlg(alg), 16)
                    try:
                        with torch.cuda.stream(stream):
                            fn(m, ys, spec, be)  # warm-up
                            torch.cuda.synchronize()
                            e0 = torch.cuda.Event(enable_timing=True)
                            e1 = torch.cuda.Event(enable_timing=True)
                            e0.record(stream)
                            for _ in range(args.reps):
                                fn(m, ys, spec, be)
                            e1.record(stream)
                        torch.cuda.synchronize()
                        ms = e0.elapsed_time(e1) / args.reps
                        rec = {"method": meth, "alg": psk.ScanAlg(alg).name, "dtype": dts,
                               "log2t": lt, "ms": round(ms, 4), "steps_per_s": T / (ms * 1e-3),
                               "launches": be.last_launch_count()}
                    except Exception as e:  # noqa: BLE001
                        rec = {"method": meth, "alg": alg, "dtype": dts, "log2t": lt,
                               "error": str(e)[:200]}
                    print(json.dumps(rec), flush=True)
            del m, ys
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
