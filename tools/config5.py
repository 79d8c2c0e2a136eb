#!/usr/bin/env python
"""BASELINE configs[4]: higher-dimensional state (nx = 16, ny = 8), T = 2^20,
a batch of B independent sequences, each with its own time-invariant model
(stride-0 broadcast fields; only y is streamed), PRTS through the wide
(warp-per-chunk) fast path.  FP64 and FP32.  Prints JSON lines: per-dtype
time-steps/s over the batch (B * T / total time, CUDA events).

Models are drawn like the reference's gen_model (model_gen.hpp:104-158):
F = 0.99 * (orthogonal factor of a Gaussian matrix), Q and R random SPD
(X X^T / n + 1e-6 I), H Gaussian, u = d = 0, prior N(0, I); y drawn from the
stationary marginal N(0, H P_inf H^T + R).  (numpy here: this is a measurement tool, the parity of the wide
path against the reference restatement is tests/test_gpu_parity.py.)

usage: python tools/config5.py [--batch 64] [--log2t 20] [--dtypes f64,f32]
                               [--how batch,loop] [--nx 16] [--ny 8]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def model(seed: int, nx: int, ny: int, t: int):
    rng = np.random.default_rng(seed)
    q_, _ = np.linalg.qr(rng.standard_normal((nx, nx)))
    F = 0.99 * q_
    X = rng.standard_normal((nx, nx))
    Q = X @ X.T / nx + 1e-6 * np.eye(nx)
    Y = rng.standard_normal((ny, ny))
    R = Y @ Y.T / ny + 1e-6 * np.eye(ny)
    H = rng.standard_normal((ny, nx))
    # measurements drawn from the stationary marginal of y (x ~ N(0, P_inf),
    # P_inf = F P_inf F^T + Q by fixed-point iteration): the timing does not
    # depend on the trajectory, and a T-step Python recursion per sequence
    # would dominate the tool's run time
    P = np.eye(nx)
    for _ in range(2000):
        P = F @ P @ F.T + Q
    Sy = H @ P @ H.T + R
    ys = rng.standard_normal((t, ny)) @ np.linalg.cholesky(Sy).T
    return F, Q, H, R, ys


def main() -> None:
    import torch

    import paper_2511_10363_b200 as psk

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--log2t", type=int, default=20)
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--nx", type=int, default=16)
    ap.add_argument("--ny", type=int, default=8)
    ap.add_argument("--how", default="batch,loop")
    args = ap.parse_args()
    T, nx, ny = 1 << args.log2t, args.nx, args.ny
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    be = psk.CudaBackend(0, mode="fast", stream=stream)
    seqs = [model(1000 + b, nx, ny, T) for b in range(args.batch)]
    for dts in args.dtypes.split(","):
        tdt = torch.float64 if dts == "f64" else torch.float32
        c = lambda a: torch.as_tensor(a, dtype=tdt, device=dev)  # noqa: E731
        ms_ = [psk.Lgssm(f=c(F), u=c(np.zeros(nx)), q=c(Q), h=c(H), d=c(np.zeros(ny)), r=c(R),
                         prior_mean=c(np.zeros(nx)), prior_cov=c(np.eye(nx)), t=T)
               for F, Q, H, R, _ in seqs]
        ys_ = [c(s[4]) for s in seqs]
        spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback)
        outs = [psk.GaussianStats(torch.empty((T, nx), dtype=tdt, device=dev),
                                  torch.empty((T, nx, nx), dtype=tdt, device=dev))
                for _ in range(args.batch)]
        with torch.cuda.stream(stream):
            psk.prts_run(ms_[0], ys_[0], spec, be, out=outs[0])  # warm-up
            psk.prts_run_batch(ms_, ys_, spec, be, outs=outs)
        torch.cuda.synchronize()
        for how in args.how.split(","):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                if how == "loop":  # one synchronous call per sequence
                    for m, ys, o in zip(ms_, ys_, outs):
                        psk.prts_run(m, ys, spec, be, out=o)
                else:  # one psk_prts_batch call (sub-streams)
                    psk.prts_run_batch(ms_, ys_, spec, be, outs=outs)
                e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            print(json.dumps({"config": f"nx={nx} ny={ny} T=2^{args.log2t} batch={args.batch} "
                                        "time-invariant models, PRTS",
                              "dtype": dts, "how": how, "ms_total": round(ms, 2),
                              "ms_per_sequence": round(ms / args.batch, 3),
                              "steps_per_s": args.batch * T / (ms * 1e-3)}), flush=True)
        del outs, ms_, ys_  # the FP64 outputs of 64 series at 2^20 hold ~146 GB
        torch.cuda.empty_cache()

if __name__ == "__main__":
    main()
