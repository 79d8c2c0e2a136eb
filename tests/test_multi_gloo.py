"""The N>1 time-sharded PRTS orchestration (distributed.py) on CPU ranks over
gloo: the same prts_sharded() the GPU ranks run, driven by an oracle-backed
shard engine, must reproduce the sequential RTS smoother of the whole series
for world sizes 2 and 3 (uneven shards).  Checks the exchange order, the
non-commutative prefix / suffix folds and the shard-boundary handling (extra
transition, prior only on rank 0, a_T only on the last rank)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _np(x):
    """numpy view of a (CPU) torch tensor the engine fills in place"""
    return x.numpy() if hasattr(x, "numpy") else x


class OracleShardEngine:
    """Reference-algorithm shard phases on the CPU (tests only)."""

    def __init__(self, orc, m, ys, lo, hi):
        import torch
        self.o, self.m, self.ys, self.lo, self.hi = orc, m, ys, lo, hi
        self.nx = m.nx
        self.torch = torch

    def _t(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a))

    def filter_reduce(self, spec):
        acc = None
        for k in range(self.lo + 1, self.hi + 1):  # 1-based steps of the shard
            e = self.o.make_filter_element(self.m, self.ys, k)
            acc = e if acc is None else self.o.filter_combine(self.nx, acc, e)
        return self._t(acc)

    def fold(self, kind, elems):
        els = [np.asarray(e) for e in elems]
        nx = self.nx
        if kind == "filter":
            acc = els[0]
            for e in els[1:]:
                acc = self.o.filter_combine(nx, acc, e)
            b, c = acc[nx * nx:nx * nx + nx], acc[nx * nx + nx:2 * nx * nx + nx]
        elif kind == "backward":
            acc = els[0]
            for e in els[1:]:
                acc = self.o.filter_combine(nx, acc, e)
            b, c = acc[2 * nx * nx + nx:2 * nx * nx + 2 * nx], acc[2 * nx * nx + 2 * nx:]
        else:
            acc = els[-1]
            for e in els[-2::-1]:
                acc = self.o.smoother_combine(nx, e, acc)
            b, c = acc[nx * nx:nx * nx + nx], acc[nx * nx + nx:]
        return self._t(np.concatenate([b, c]))

    def stats(self, t):
        return (self.torch.zeros((t, self.nx), dtype=self.torch.float64),
                self.torch.zeros((t, self.nx, self.nx), dtype=self.torch.float64))

    def _slice(self, prior=None):
        from paper_2511_10363_b200.api import Lgssm
        s = slice(self.lo, self.hi)
        m = self.m
        pm, pc = (m.prior_mean, m.prior_cov) if prior is None else prior
        return Lgssm(f=m.f[s], u=m.u[s], q=m.q[s], h=m.h[s], d=m.d[s], r=m.r[s],
                     prior_mean=pm, prior_cov=pc, t=self.hi - self.lo), self.ys[s]

    def filter_finish(self, carry, mean, cov):
        nx = self.nx
        prior = None
        if carry is not None:
            c = np.asarray(carry)
            prior = (c[:nx].copy(), c[nx:].reshape(nx, nx).copy())
        sm, sys_ = self._slice(prior)
        fm, fc = self.o.kf_run(sm, sys_)
        _np(mean)[:], _np(cov)[:] = fm, fc

    def smoother_reduce(self, spec, mean, cov):
        mean, cov = _np(mean), _np(cov)
        acc = None
        for i in range(self.hi - 1, self.lo - 1, -1):
            e = self.o.make_smoother_element(self.m, self.ys, mean[i - self.lo],
                                             cov[i - self.lo], i + 1)
            acc = e if acc is None else self.o.smoother_combine(self.nx, e, acc)
        return self._t(acc)

    # ---- the backward half of a sharded PTFS (kalman_par.hpp:63-89, 183-201)
    def _shifted(self, j):
        """slot j (0-based) holds a(step j+1): make_filter_element with the
        1-based step j + 2; identity past the series' last transition."""
        nx = self.nx
        if j + 1 < int(self.m.t):
            return self.o.make_filter_element(self.m, self.ys, j + 2)
        e = np.zeros(3 * nx * nx + 2 * nx)
        e[:nx * nx] = np.eye(nx).ravel()
        return e

    def backward_reduce(self, spec):
        acc = None
        for j in range(self.lo, self.hi):
            e = self._shifted(j)
            acc = e if acc is None else self.o.filter_combine(self.nx, acc, e)
        return self._t(acc)

    def backward_finish(self, carry, fmean, fcov, mean, cov):
        nx = self.nx
        state = None
        if carry is not None:  # (eta, J) only: an identity element carrying them
            c = np.asarray(carry)
            state = np.zeros(3 * nx * nx + 2 * nx)
            state[:nx * nx] = np.eye(nx).ravel()
            state[2 * nx * nx + nx:2 * nx * nx + 2 * nx] = c[:nx]
            state[2 * nx * nx + 2 * nx:] = c[nx:]
        fm, fc = _np(fmean), _np(fcov)
        mean, cov = _np(mean), _np(cov)
        for j in range(self.hi - 1, self.lo - 1, -1):
            e = self._shifted(j)
            state = e if state is None else self.o.filter_combine(nx, e, state)
            eta = state[2 * nx * nx + nx:2 * nx * nx + 2 * nx].copy()
            jm = state[2 * nx * nx + 2 * nx:].reshape(nx, nx).copy()
            x, p = self.o.tf_combine(fm[j - self.lo].copy(), fc[j - self.lo].copy(), eta, jm)
            mean[j - self.lo], cov[j - self.lo] = x, p

    def smoother_finish(self, carry, mean, cov):
        nx = self.nx
        mean, cov = _np(mean), _np(cov)
        state = None
        if carry is not None:
            c = np.asarray(carry)
            state = np.concatenate([np.zeros(nx * nx), c])  # (E=0, g, L)
        for i in range(self.hi - 1, self.lo - 1, -1):
            e = self.o.make_smoother_element(self.m, self.ys, mean[i - self.lo],
                                             cov[i - self.lo], i + 1)
            state = e if state is None else self.o.smoother_combine(nx, e, state)
            mean[i - self.lo] = state[nx * nx:nx * nx + nx]
            cov[i - self.lo] = state[nx * nx + nx:].reshape(nx, nx)


def _worker(rank, world, port, t, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist

    from conftest import gen
    from oracle.oracle import Oracle
    from paper_2511_10363_b200.api import ScanSpec
    from paper_2511_10363_b200.distributed import prts_sharded, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("port")
    m, ys = gen(orc, 12, 4, 2, t)
    lo, hi = shard_range(t, rank, world)
    eng = OracleShardEngine(orc, m, ys, lo, hi)
    mean, cov = prts_sharded(eng, ScanSpec(), rank, world, hi - lo)
    np.savez(Path(out_dir) / f"r{rank}.npz", mean=mean, cov=cov, lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


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


@pytest.mark.parametrize("world,t", [(2, 101), (3, 64)])
def test_sharded_prts_matches_sequential(tmp_path, port, world, t):
    import torch.multiprocessing as mp

    from conftest import gen, max_rel_err
    _spawn(_worker, world, t, str(tmp_path))
    m, ys = gen(port, 12, 4, 2, t)
    rm, rc = port.rts_run(m, ys)
    covered = 0
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        lo, hi = int(d["lo"]), int(d["hi"])
        assert lo == covered
        covered = hi
        assert max_rel_err(d["mean"], d["cov"], rm[lo:hi], rc[lo:hi]) < 1e-9, r
    assert covered == t


def test_shard_range_partition():
    from paper_2511_10363_b200.distributed import shard_range
    for t in (1, 7, 64, 1000):
        for w in (1, 2, 3, 8):
            spans = [shard_range(t, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == t
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_shard_model_slices_with_boundary_transition():
    """distributed.shard_model: per-step fields cover [lo, hi + 1) (the
    smoother boundary transition) except on the last shard; time-invariant
    fields stay one block; the prior is passed through."""
    import torch

    from paper_2511_10363_b200.api import Lgssm
    from paper_2511_10363_b200.distributed import shard_model
    t = 10
    f = np.arange(t * 4, dtype=np.float64).reshape(t, 2, 2)
    m = Lgssm(f=f, u=np.zeros(2), q=np.eye(2), h=np.ones((t, 1, 2)), d=np.zeros(1),
              r=np.eye(1), prior_mean=np.zeros(2), prior_cov=np.eye(2), t=t)
    ys = np.arange(t, dtype=np.float64).reshape(t, 1)
    ms, yss = shard_model(m, ys, 3, 6)
    assert ms.t == 4 and tuple(ms.f.shape) == (4, 2, 2) and tuple(ms.h.shape) == (4, 1, 2)
    assert torch.equal(ms.f, torch.as_tensor(f[3:7]))
    assert tuple(ms.u.shape) == (2,) and tuple(ms.q.shape) == (2, 2)
    assert torch.equal(yss, torch.as_tensor(ys[3:7]))
    ml, ysl = shard_model(m, ys, 6, 10)  # last shard: no extra transition
    assert ml.t == 4 and torch.equal(ml.f, torch.as_tensor(f[6:10]))
    m32, _ = shard_model(m, ys, 0, 5, dtype=torch.float32)
    assert m32.f.dtype == torch.float32



def _ptfs_worker(rank, world, port, t, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist

    from conftest import gen
    from oracle.oracle import Oracle
    from paper_2511_10363_b200.api import ScanSpec
    from paper_2511_10363_b200.distributed import (ptfs_groups, ptfs_halves, ptfs_sharded,
                                                   shard_range)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    groups = ptfs_groups(world)
    orc = Oracle("port")
    m, ys = gen(orc, 14, 4, 2, t)
    fwd, i, h = ptfs_halves(rank, world)
    lo, hi = shard_range(t, i, h)
    eng = OracleShardEngine(orc, m, ys, lo, hi)
    out = ptfs_sharded(eng, ScanSpec(), rank, world, hi - lo, groups)
    if out is not None:
        np.savez(Path(out_dir) / f"p{i}.npz", mean=np.asarray(out[0]), cov=np.asarray(out[1]),
                 lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,t", [(2, 37), (4, 61), (6, 50)])
def test_sharded_ptfs_halves_matches_rts(tmp_path, port, world, t):
    """PTFS with the forward filter time-sharded over ranks [0, G/2) and the
    backward filter over [G/2, G) (distributed.ptfs_sharded) reproduces the
    sequential RTS smoother (the reference checks ptfs against rts_run at
    1e-9, test_kalman_par.cpp:209-227)."""
    import torch.multiprocessing as mp

    from conftest import gen, max_rel_err
    _spawn(_ptfs_worker, world, t, str(tmp_path))
    m, ys = gen(port, 14, 4, 2, t)
    rm, rc = port.rts_run(m, ys)
    covered = 0
    for i in range(world // 2):
        d = np.load(tmp_path / f"p{i}.npz")
        lo, hi = int(d["lo"]), int(d["hi"])
        assert lo == covered
        covered = hi
        assert max_rel_err(d["mean"], d["cov"], rm[lo:hi], rc[lo:hi]) < 1e-9, i
    assert covered == t
