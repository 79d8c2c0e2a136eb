#!/usr/bin/env python
"""BASELINE configs[4]: higher-dimensional state (nx = 16, ny = 8), T = 2^20,
a batch of B independent sequences, each with its own time-invariant model
(stride-0 broadcast fields; only y is streamed), PRTS through the fast path
for dims > 4 (register-tiled warp kernels, psk_tile_impl.cuh; `--tile 0`:
the runtime-dimension warp kernels for an A/B).  FP64 and FP32.  Prints JSON
lines: per-dtype time-steps/s over the batch (B * T / total time, CUDA events).

Inputs as SURVEY.md 8(d) item 3 specifies: series b is the reference's
gen_model(seed + b, 16, 8, 1) broadcast over T, y = simulate_data on that
model over T steps (seed + b + 1) -- drawn with the reference restatement in
oracle/ (input generation only; parity of these series is
tests/test_gpu_headline.py::test_config5_subset_2p20_f64).

usage: python tools/config5.py [--batch 64] [--log2t 20] [--dtypes f64,f32]
                               [--how batch,loop] [--tile 1]
"""
from __future__ import annotations

import argparse
import json
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def model(orc, seed: int, b: int, nx: int, ny: int, t: int):
    g = orc.gen_model(seed + b, nx, ny, 1)
    blk = {k: g[k][0] for k in ("f", "u", "q", "h", "d", "r")}
    gt = dict(blk, m0=g["m0"], p0=g["p0"], t=t, nx=nx, ny=ny, bcast=0x3F)
    ys = orc.simulate_data(gt, seed + b + 1)
    return blk, g["m0"], g["p0"], ys


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
    ap.add_argument("--tile", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--waves", type=int, default=0, help="auto chunk: waves of chunks (0: default)")
    ap.add_argument("--method", default="prts", choices=["prts", "pkf", "ptfs"],
                    help="ptfs runs one call per sequence (no batch entry point)")
    args = ap.parse_args()
    from oracle.oracle import Oracle  # the reference's generator (inputs only)
    T, nx, ny = 1 << args.log2t, args.nx, args.ny
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    be = psk.CudaBackend(0, mode="fast", stream=stream)
    be.set_option("tile", args.tile)
    if args.waves:
        be.set_option("waves", args.waves)
    orc = Oracle("port")
    with ThreadPoolExecutor(16) as ex:
        seqs = list(ex.map(lambda b: model(orc, args.seed, b, nx, ny, T), range(args.batch)))
    for dts in args.dtypes.split(","):
        tdt = torch.float64 if dts == "f64" else torch.float32
        c = lambda a: torch.as_tensor(a, dtype=tdt, device=dev)  # noqa: E731
        ms_ = [psk.Lgssm(**{k: c(v) for k, v in blk.items()}, prior_mean=c(m0),
                         prior_cov=c(p0), t=T)
               for blk, m0, p0, _ in seqs]
        ys_ = [c(s[3]) for s in seqs]
        spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback)
        outs = [psk.GaussianStats(torch.empty((T, nx), dtype=tdt, device=dev),
                                  torch.empty((T, nx, nx), dtype=tdt, device=dev))
                for _ in range(args.batch)]
        single = {"prts": psk.prts_run, "pkf": psk.pkf_run, "ptfs": psk.ptfs_run}[args.method]
        batch = {"prts": psk.prts_run_batch, "pkf": psk.pkf_run_batch}.get(args.method)
        with torch.cuda.stream(stream):
            single(ms_[0], ys_[0], spec, be, out=outs[0])  # warm-up
            if batch is not None:
                batch(ms_, ys_, spec, be, outs=outs)
        torch.cuda.synchronize()
        for how in args.how.split(","):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                if how == "loop" or batch is None:  # one synchronous call per sequence
                    how = "loop"
                    for m, ys, o in zip(ms_, ys_, outs):
                        single(m, ys, spec, be, out=o)
                else:  # one psk_prts_batch / psk_pkf_batch call (sub-streams)
                    batch(ms_, ys_, spec, be, outs=outs)
                e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            print(json.dumps({"config": f"nx={nx} ny={ny} T=2^{args.log2t} batch={args.batch} "
                                        f"time-invariant gen_model models, {args.method.upper()}",
                              "tile": args.tile, "waves": args.waves,
                              "dtype": dts, "how": how, "ms_total": round(ms, 2),
                              "ms_per_sequence": round(ms / args.batch, 3),
                              "steps_per_s": args.batch * T / (ms * 1e-3)}), flush=True)
        del outs, ms_, ys_  # the FP64 outputs of 64 series at 2^20 hold ~146 GB
        torch.cuda.empty_cache()

if __name__ == "__main__":
    main()
