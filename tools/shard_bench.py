#!/usr/bin/env python
"""Per-rank cost of the time-sharded PRTS (BASELINE configs[3]) on ONE GPU:
the phases of a middle rank of G over its T/G-step shard, the all_gathers
replaced by local stand-ins (NCCL needs one GPU per rank), against the plain
single-GPU PRTS of the same T/G steps.  Shows the sharding overhead the
scaling run pays on top of the ideal T/G work.  Prints JSON lines.

usage: python tools/shard_bench.py [log2T=24] [G list=2,4,8]
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
    from paper_2511_10363_b200.distributed import CudaShardEngine, prts_sharded, shard_range
    from paper_2511_10363_b200.synthetic import cv_matrices, simulate_cv

    log2t = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    Gs = [int(g) for g in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
    T = 1 << log2t
    F, Q, H, R, m0, P0 = cv_matrices()
    dev = torch.device("cuda", 0)
    ys_all = simulate_cv(T, seed=0)

    def model(n):
        f = lambda a: torch.as_tensor(a, dtype=torch.float64, device=dev).expand(  # noqa: E731
            n, *np.shape(a)).contiguous()
        return psk.Lgssm(f=f(F), u=f(np.zeros(4)), q=f(Q), h=f(H), d=f(np.zeros(2)), r=f(R),
                         prior_mean=torch.as_tensor(m0, device=dev),
                         prior_cov=torch.as_tensor(P0, device=dev), t=n)

    spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback)
    for G in Gs:
        rank = 1 if G > 2 else 0
        lo, hi = shard_range(T, rank, G)
        n_in = hi + 1 - lo
        m = model(n_in)
        ys = torch.as_tensor(ys_all[lo:hi + 1], device=dev)
        be = psk.CudaBackend(0)
        be.set_option("async", 1)  # as bench.py's timed region
        from paper_2511_10363_b200.distributed import shard_flags
        eng = CudaShardEngine(be, m, ys, shard_flags(rank, G), hi - lo)

        def gather_stub(x, world, group=None):
            return [x] * world

        import paper_2511_10363_b200.distributed as D
        real = D.all_gather
        D.all_gather = gather_stub
        try:
            def step():
                return prts_sharded(eng, spec, rank, G, hi - lo)

            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms_shard = e0.elapsed_time(e1) / reps
        finally:
            D.all_gather = real
        # plain PRTS of the same number of steps
        mp = model(hi - lo)
        ysp = torch.as_tensor(ys_all[lo:hi], device=dev)
        bp = psk.CudaBackend(0)
        bp.set_option("async", 1)
        bp.set_stream(torch.cuda.current_stream())  # the events' stream
        for _ in range(3):
            psk.prts_run(mp, ysp, spec, bp)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            psk.prts_run(mp, ysp, spec, bp)
        e1.record()
        torch.cuda.synchronize()
        ms_plain = e0.elapsed_time(e1) / 10
        print(json.dumps({"T": f"2^{log2t}", "G": G, "shard_steps": hi - lo,
                          "rank_phases_ms": round(ms_shard, 4),
                          "plain_prts_same_steps_ms": round(ms_plain, 4),
                          "overhead_ms": round(ms_shard - ms_plain, 4)}), flush=True)
        del m, ys, mp, ysp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
