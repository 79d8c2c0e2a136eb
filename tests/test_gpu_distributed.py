"""The multi-process time-sharded PRTS exactly as bench.py runs it -- the real
distributed.prts_run_sharded with the CUDA shard engine (CudaShardEngine,
shard_async on torch's stream) and a real torch.distributed all_gather -- in
2 and 3 processes that share the one GPU of the test box (NCCL refuses two
ranks on one device, so the collective is gloo on CUDA tensors here; the bench
uses NCCL over NVLink).  The concatenated shard outputs must match the CPU
oracle's sequential rts_run over all T = 2^20 steps at the FP64 gate
(kalman_par.hpp:156-179 prts_run vs kalman_seq.hpp rts_run)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import max_rel_err

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
T = 1 << 20


def _worker(rank, world, port, out_dir, alg):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200 import distributed as dp
    from paper_2511_10363_b200.synthetic import cv_model

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    m, ys = cv_model(T, seed=21)
    lo, hi = dp.shard_range(T, rank, world)
    ms, yss = dp.shard_model(m, ys, lo, hi, device=dev)
    be = psk.CudaBackend(0, mode="fast")
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        out = dp.prts_run_sharded(ms, yss, psk.ScanSpec(psk.ScanAlg(alg), 16), be, rank,
                                  world, lo, hi, T, dist.group.WORLD)
    torch.cuda.synchronize()
    np.savez(Path(out_dir) / f"r{rank}.npz", mean=out.mean.cpu().numpy(),
             cov=out.cov.cpu().numpy(), lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *rest):
    """mp.spawn with a fresh rendezvous port; retried when another process
    took the port between _free_port() and the bind (EADDRINUSE)."""
    import torch.multiprocessing as mp
    for attempt in range(3):
        try:
            mp.spawn(fn, args=(world, _free_port(), *rest), nprocs=world, join=True)
            return
        except Exception as e:  # noqa: BLE001
            msg = str(e)
            if attempt == 2 or ("Address already in use" not in msg and "EADDRINUSE" not in msg):
                raise


@pytest.fixture(scope="module")
def rts_ref(port):
    from paper_2511_10363_b200.synthetic import cv_model
    m, ys = cv_model(T, seed=21)
    return port.rts_run(m, ys)


@pytest.mark.parametrize("world,alg", [(2, 6), (3, 3)])
def test_prts_run_sharded_processes(gpu, tmp_path, rts_ref, world, alg):
    import torch.multiprocessing as mp

    _spawn(_worker, world, str(tmp_path), alg)
    rm, rc = rts_ref
    covered = 0
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        lo, hi = int(d["lo"]), int(d["hi"])
        assert lo == covered
        covered = hi
        e = max_rel_err(d["mean"], d["cov"], rm[lo:hi], rc[lo:hi])
        assert e < 1e-9, (r, e)
    assert covered == T


def _batch_worker(rank, world, port, out_dir):
    """BASELINE configs[4]'s multi-GPU form: batch sharding, no exchange --
    each rank runs its contiguous share of the series through one
    psk_prts_batch call (distributed.prts_run_batch_sharded)."""
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200 import distributed as dp
    from oracle.oracle import Oracle
    from test_gpu_headline import _config5_series

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("port")
    series = [_config5_series(orc, psk, b, 2048) for b in range(5)]
    be = psk.CudaBackend(0)
    idx, res = dp.prts_run_batch_sharded([s[0] for s in series], [s[1] for s in series],
                                         psk.ScanSpec(psk.ScanAlg.DecoupledLookback), be,
                                         rank, world)
    np.savez(Path(out_dir) / f"b{rank}.npz", idx=np.array(list(idx)),
             **{f"m{i}": r.mean for i, r in zip(idx, res)},
             **{f"c{i}": r.cov for i, r in zip(idx, res)})
    dist.barrier()
    dist.destroy_process_group()


def test_config5_batch_sharded_processes(gpu, tmp_path, port):
    import torch.multiprocessing as mp

    import paper_2511_10363_b200 as psk
    from test_gpu_headline import _config5_series

    world = 2
    _spawn(_batch_worker, world, str(tmp_path))
    seen = []
    for r in range(world):
        d = np.load(tmp_path / f"b{r}.npz")
        for i in d["idx"]:
            m, ys = _config5_series(port, psk, int(i), 2048)
            rm, rc = port.rts_run(m, ys)
            e = max_rel_err(d[f"m{i}"], d[f"c{i}"], rm, rc)
            assert e < 1e-9, (r, int(i), e)
            seen.append(int(i))
    assert sorted(seen) == list(range(5))  # every series exactly once


def _ptfs_worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200 import distributed as dp
    from paper_2511_10363_b200.synthetic import cv_model

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    groups = dp.ptfs_groups(world)
    dev = torch.device("cuda", 0)
    m, ys = cv_model(T, seed=23)
    fwd, i, h = dp.ptfs_halves(rank, world)
    lo, hi = dp.shard_range(T, i, h)
    ms, yss = dp.shard_model(m, ys, lo, hi, device=dev)
    be = psk.CudaBackend(0)
    out = dp.ptfs_run_sharded(ms, yss, psk.ScanSpec(psk.ScanAlg.DecoupledLookback, 16), be,
                              rank, world, lo, hi, groups)
    torch.cuda.synchronize()
    if out is not None:
        np.savez(Path(out_dir) / f"p{i}.npz", mean=out.mean.cpu().numpy(),
                 cov=out.cov.cpu().numpy(), lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ptfs_halves_processes(gpu, tmp_path, port, world):
    """configs[2] shape: the two-filter smoother with the forward filter on
    one half of the ranks and the backward filter on the other (each half
    time-sharded), real processes and collectives, T = 2^20, vs rts_run."""
    import torch.multiprocessing as mp

    from paper_2511_10363_b200.synthetic import cv_model
    _spawn(_ptfs_worker, world, str(tmp_path))
    m, ys = cv_model(T, seed=23)
    rm, rc = port.rts_run(m, ys)
    covered = 0
    for i in range(world // 2):
        d = np.load(tmp_path / f"p{i}.npz")
        lo, hi = int(d["lo"]), int(d["hi"])
        assert lo == covered
        covered = hi
        e = max_rel_err(d["mean"], d["cov"], rm[lo:hi], rc[lo:hi])
        assert e < 1e-9, (i, e)
    assert covered == T
