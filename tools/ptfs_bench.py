#!/usr/bin/env python
"""BASELINE configs[2]: parallel two-filter smoother, T = 2^20 (damped CV,
nx = 4, ny = 2, FP64, device-resident): PTFS on one context vs forward and
backward passes on two contexts (devices = 2: two GPUs when more than one is
visible, else two streams of one GPU), next to PRTS.  CUDA events around the
synchronous calls (the two-context call spans both devices, so its time is
taken on the forward device after both finished); the multi-device context
(psk_create_multi over all visible GPUs, or two streams of GPU 0) runs the
two filters on its halves.  Prints JSON lines.
"""
from __future__ import annotations

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

    log2t = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    T = 1 << log2t
    ngpu = torch.cuda.device_count()
    F, Q, H, R, m0, P0 = cv_matrices()
    dev = torch.device("cuda", 0)

    def field(a):
        t = torch.as_tensor(a, dtype=torch.float64, device=dev)
        return t.expand(T, *t.shape).contiguous()

    m = psk.Lgssm(f=field(F), u=field(np.zeros(4)), q=field(Q), h=field(H),
                  d=field(np.zeros(2)), r=field(R),
                  prior_mean=torch.as_tensor(m0, device=dev),
                  prior_cov=torch.as_tensor(P0, device=dev), t=T)
    ys = torch.as_tensor(simulate_cv(T, seed=3), device=dev)
    fwd = psk.CudaBackend(0)
    bwd = psk.CudaBackend(1 if ngpu > 1 else 0)
    spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback)
    # a multi-device context (psk_create_multi): the two filters on its two
    # halves, each time-sharded when the halves have several devices
    devs = list(range(min(ngpu, 8))) if ngpu > 1 else [0, 0]
    multi = psk.CudaBackend(devs)
    runs = {"prts": lambda: psk.prts_run(m, ys, spec, fwd),
            "ptfs_1ctx": lambda: psk.ptfs_run(m, ys, spec, fwd),
            "ptfs_2ctx": lambda: psk.ptfs_run(m, ys, spec, fwd, bwd, 2),
            "ptfs_multi": lambda: psk.ptfs_run(m, ys, spec, multi, multi, len(devs)),
            "prts_multi": lambda: psk.prts_run(m, ys, spec, multi)}
    for name, fn in runs.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"config": f"T=2^{log2t} nx=4 ny=2 f64", "run": name,
                          "bwd_device": bwd.device if name == "ptfs_2ctx" else None,
                          "devices": devs if name.endswith("multi") else None,
                          "ms": round(ms, 4), "steps_per_s": T / (ms * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
