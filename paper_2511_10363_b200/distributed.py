"""Multi-GPU time sharding of the parallel RTS smoother.

One process per GPU.  Rank g owns the contiguous steps [lo, hi) of the series
(plus one extra transition (F, Q, u) for the smoother boundary).  The only
data-path exchanges are two tiny all_gathers of shard elements -- one
filtering element (3 nx^2 + 2 nx scalars) and one smoothing element
(2 nx^2 + nx) per rank, NCCL over NVLink on the GPU box:

  1. filter reduce+scan on the shard        -> shard element a_g
  2. all_gather(a_0 .. a_{G-1})
  3. carry_g = a_0 (x) ... (x) a_{g-1}       (non-commutative, rank order; a_0
                                              contains a_1 with A = 0, so the
                                              fold is the filtered state at lo-1)
  4. filter finish from carry_g             -> filtered stats of the shard
  5. smoother reduce+scan                   -> shard suffix element s_g
  6. all_gather(s_0 .. s_{G-1})
  7. carry'_g = s_{g+1} (x) ... (x) s_{G-1}  (s_{G-1} contains a_T with E = 0:
                                              the smoothed state at hi)
  8. smoother finish from carry'_g          -> smoothed stats of the shard

The fix-up is not a separate pass: the carried state enters the finish
kernels that write the outputs anyway.  `prts_run_sharded` is written against
a small engine interface so that the same orchestration runs on the CUDA
engine (product) and, in the CPU tests, on an oracle-backed engine over gloo.
"""
from __future__ import annotations

import ctypes as C
from typing import Any

from . import _lib


def shard_range(t: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous near-equal split of [0, t) (earlier ranks get the remainder)."""
    base, rem = divmod(t, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


class CudaShardEngine:
    """Shard phases on one GPU through the C-ABI (psk_shard_*, psk_fold_*)."""

    def __init__(self, be, model, ys, flags: int, t_shard: int):
        from .api import _Marshal
        self.be = be
        self.mk = _Marshal(model, ys)
        if self.mk.device is None:
            raise ValueError("sharded runs take CUDA tensors")
        self.mk.model.t = t_shard  # f/u/q may hold one extra transition
        self.mk.t = t_shard
        self.flags = flags
        self.nx = self.mk.nx
        import torch
        self.torch = torch
        # the phases, the element all_gathers (NCCL, torch's current stream)
        # and the folds are queued back to back on one stream without host
        # synchronisation; the smoother finish synchronises and reports errors
        be.set_stream(torch.cuda.current_stream(self.mk.device))
        be.set_option("shard_async", 1)
        self.dt = torch.float64 if self.mk.f64 else torch.float32
        self.dev = self.mk.device

    def _p(self, t):
        return C.c_void_p(t.data_ptr() if t is not None else 0)

    def empty(self, n):
        return self.torch.empty(n, dtype=self.dt, device=self.dev)

    def filter_reduce(self, spec):
        from .api import _check
        out = self.empty(3 * self.nx * self.nx + 2 * self.nx)
        _check(_lib.lib().psk_shard_filter_reduce(self.be.handle, C.byref(self.mk.model),
                                                  self.flags, int(spec.alg),
                                                  int(spec.sengupta_n), self._p(out)))
        return out

    def filter_finish(self, carry, mean, cov):
        from .api import _check
        _check(_lib.lib().psk_shard_filter_finish(self.be.handle, C.byref(self.mk.model),
                                                  self.flags, self._p(carry), self._p(mean),
                                                  self._p(cov)))

    def smoother_reduce(self, spec, mean, cov):
        from .api import _check
        out = self.empty(2 * self.nx * self.nx + self.nx)
        _check(_lib.lib().psk_shard_smoother_reduce(self.be.handle, C.byref(self.mk.model),
                                                    self.flags, int(spec.alg),
                                                    int(spec.sengupta_n), self._p(mean),
                                                    self._p(cov), self._p(out)))
        return out

    def smoother_finish(self, carry, mean, cov):
        from .api import _check
        _check(_lib.lib().psk_shard_smoother_finish(self.be.handle, C.byref(self.mk.model),
                                                    self.flags, self._p(carry), self._p(mean),
                                                    self._p(cov)))

    def backward_reduce(self, spec):
        """PTFS backward half: shifted elements of the shard + reverse scan;
        returns the shard's backward total (a filter element)."""
        from .api import _check
        out = self.empty(3 * self.nx * self.nx + 2 * self.nx)
        _check(_lib.lib().psk_shard_backward_reduce(self.be.handle, C.byref(self.mk.model),
                                                    self.flags, int(spec.alg),
                                                    int(spec.sengupta_n), self._p(out)))
        return out

    def backward_finish(self, carry, fmean, fcov, mean, cov):
        from .api import _check
        _check(_lib.lib().psk_shard_backward_finish(self.be.handle, C.byref(self.mk.model),
                                                    self.flags, self._p(carry), self._p(fmean),
                                                    self._p(fcov), self._p(mean), self._p(cov)))

    def fold(self, kind: str, elems):
        from .api import _check
        st = self.empty(self.nx + self.nx * self.nx)
        stacked = self.torch.stack(list(elems)).contiguous()
        fn = {"filter": _lib.lib().psk_fold_filter, "smoother": _lib.lib().psk_fold_smoother,
              "backward": _lib.lib().psk_fold_backward}[kind]
        _check(fn(self.be.handle, _lib.PSK_F64 if self.mk.f64 else _lib.PSK_F32, self.nx,
                  self._p(stacked), len(elems), self._p(st)))
        return st

    def stats(self, t):
        return (self.torch.empty((t, self.nx), dtype=self.dt, device=self.dev),
                self.torch.empty((t, self.nx, self.nx), dtype=self.dt, device=self.dev))


def all_gather(x, world: int, group: Any = None):
    import torch.distributed as dist
    out = [x.new_empty(x.shape) for _ in range(world)]
    dist.all_gather(out, x, group=group)
    return out


def prts_sharded(engine, spec, rank: int, world: int, t_shard: int, group: Any = None):
    """Steps 1-8 above on one rank; returns the shard's smoothed (mean, cov)."""
    a = engine.filter_reduce(spec)
    gathered = all_gather(a, world, group) if world > 1 else [a]
    carry = engine.fold("filter", gathered[:rank]) if rank > 0 else None
    mean, cov = engine.stats(t_shard)
    engine.filter_finish(carry, mean, cov)
    s = engine.smoother_reduce(spec, mean, cov)
    gathered = all_gather(s, world, group) if world > 1 else [s]
    carry = engine.fold("smoother", gathered[rank + 1:]) if rank < world - 1 else None
    engine.smoother_finish(carry, mean, cov)
    return mean, cov


def shard_model(model, ys, lo: int, hi: int, device: Any = None, dtype: Any = None):
    """The shard [lo, hi) of a T-step model as device tensors: per-step fields
    sliced to [lo, min(hi + 1, T)) -- f/u/q carry the one extra transition the
    smoother boundary needs, h/d/r/y the matching steps (the extra step is
    never read as a measurement) -- and time-invariant fields kept as one
    block.  Returns (Lgssm, ys)."""
    import numpy as np
    import torch

    from .api import Lgssm

    t = int(model.t)
    hi_in = min(hi + 1, t)
    nx, ny = model.nx, model.ny
    shapes = {"f": (nx, nx), "u": (nx,), "q": (nx, nx), "h": (ny, nx), "d": (ny,),
              "r": (ny, ny)}

    def put(a, shp=None):
        x = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
        if shp is not None and tuple(x.shape) != shp:  # per-step field
            x = x[lo:hi_in]
        x = x.to(device=device, dtype=dtype or x.dtype).contiguous()
        return x

    fields = {k: put(getattr(model, k), shp) for k, shp in shapes.items()}
    m = Lgssm(**fields, prior_mean=put(model.prior_mean), prior_cov=put(model.prior_cov),
              t=hi_in - lo)
    y = ys if isinstance(ys, torch.Tensor) else torch.as_tensor(np.asarray(ys))
    return m, put(y[lo:hi_in])


def ptfs_halves(rank: int, world: int) -> tuple[bool, int, int]:
    """(forward?, shard index, shards per half) of a rank of the sharded PTFS:
    ranks [0, G/2) run the forward filter, [G/2, G) the backward filter, rank
    r and r + G/2 own the same step range (PAPER.md:883-892 with each half
    time-sharded)."""
    if world < 2 or world % 2:
        raise ValueError("the two-filter smoother splits an even number of ranks in halves")
    h = world // 2
    return rank < h, rank % h, h


def ptfs_groups(world: int):
    """The two half groups (every rank must create both, in this order)."""
    import torch.distributed as dist
    h = world // 2
    return dist.new_group(list(range(h))), dist.new_group(list(range(h, world)))


def ptfs_sharded(engine, spec, rank: int, world: int, t_shard: int, groups=None):
    """The parallel two-filter smoother (Alg. 7, kalman_par.hpp:207-238) on
    disjoint GPU halves, each half time-sharded:

      forward rank i:   sharded PKF of shard i (all_gather of shard elements in
                        the forward group, prefix fold, finish) -> filtered
                        stats, sent to backward rank h + i (20 scalars / step
                        at nx = 4: the only per-step data that crosses GPUs);
      backward rank i:  shifted elements + reverse scan of shard i,
                        all_gather of the shard totals in the backward group,
                        fold of the LATER shards -> (eta, J) carry, then the
                        backward finish fused with the two-filter combination
                        over the received filtered stats -> smoothed stats.

    The two halves run concurrently.  Returns the smoothed (mean, cov) of the
    shard on backward ranks, None on forward ranks.  `engine` is a
    CudaShardEngine (forward ranks built with PSK_SHARD_FILTERED) or a test
    double with the same methods."""
    import torch.distributed as dist

    fwd, i, h = ptfs_halves(rank, world)
    gf, gb = groups if groups is not None else (None, None)
    if fwd:
        a = engine.filter_reduce(spec)
        gathered = all_gather(a, h, gf) if h > 1 else [a]
        carry = engine.fold("filter", gathered[:i]) if i > 0 else None
        mean, cov = engine.stats(t_shard)
        engine.filter_finish(carry, mean, cov)
        _p2p(dist.send, mean, h + i)
        _p2p(dist.send, cov, h + i)
        return None
    s = engine.backward_reduce(spec)
    gathered = all_gather(s, h, gb) if h > 1 else [s]
    carry = engine.fold("backward", gathered[i + 1:]) if i < h - 1 else None
    fmean, fcov = engine.stats(t_shard)
    _p2p(dist.recv, fmean, i)
    _p2p(dist.recv, fcov, i)
    mean, cov = engine.stats(t_shard)
    engine.backward_finish(carry, fmean, fcov, mean, cov)
    return mean, cov


def _p2p(op, t, peer: int) -> None:
    """Point-to-point send / recv of `t`: NCCL moves device tensors directly
    (NVLink); gloo (the CPU test rig) only moves host tensors, so a device
    tensor is staged through host memory there."""
    import torch.distributed as dist
    if dist.get_backend() == "gloo" and getattr(t, "is_cuda", False):
        h = t.cpu()
        op(h, peer)
        if op is dist.recv:
            t.copy_(h)
        return
    op(t, peer)


def ptfs_flags(rank: int, world: int) -> int:
    """Shard flags of a sharded-PTFS rank (its half's shard position)."""
    fwd, i, h = ptfs_halves(rank, world)
    f = shard_flags(i, h)
    return f | (_lib.PSK_SHARD_FILTERED if fwd else 0)


def ptfs_run_sharded(model, ys, spec, be, rank: int, world: int, lo: int, hi: int,
                     groups=None, engine: Any = None):
    """PTFS over shard [lo, hi) (shard_range(T, rank % (world/2), world/2)) on
    one rank of the two halves; `model`/`ys` hold the shard's steps plus one
    extra step of every field unless hi == T (shard_model).  Returns the
    smoothed GaussianStats of the shard on backward ranks, None on forward
    ranks."""
    from . import api

    if engine is None:
        engine = CudaShardEngine(be, model, ys, ptfs_flags(rank, world), hi - lo)
    out = ptfs_sharded(engine, spec, rank, world, hi - lo, groups)
    return None if out is None else api.GaussianStats(*out)


def shard_flags(rank: int, world: int) -> int:
    return (_lib.PSK_SHARD_FIRST if rank == 0 else 0) | \
        (_lib.PSK_SHARD_LAST if rank == world - 1 else 0)


def prts_run_sharded(model, ys, spec, be, rank: int, world: int, lo: int, hi: int,
                     t_total: int, group: Any = None, engine: Any = None):
    """PRTS over the shard [lo, hi) of a T-step series.  `model`/`ys` hold the
    shard's steps (f/u/q with one extra transition unless hi == T).  world == 1
    is the plain single-GPU prts_run."""
    from . import api

    if world == 1:
        return api.prts_run(model, ys, spec, be)
    if engine is None:
        engine = CudaShardEngine(be, model, ys, shard_flags(rank, world), hi - lo)
    mean, cov = prts_sharded(engine, spec, rank, world, hi - lo, group)
    return api.GaussianStats(mean, cov)


def batch_shard(n: int, rank: int, world: int) -> range:
    """BASELINE configs[4] on G GPUs: batch sharding -- rank
    g runs the contiguous near-equal share of the n independent series; there
    is no data-path exchange, so scaling is "weak" per series."""
    lo, hi = shard_range(n, rank, world)
    return range(lo, hi)


def prts_run_batch_sharded(models, ys_list, spec, be, rank: int, world: int):
    """This rank's share of a batch through one psk_prts_batch call; returns
    (indices, results)."""
    from . import api

    idx = batch_shard(len(models), rank, world)
    res = api.prts_run_batch([models[i] for i in idx], [ys_list[i] for i in idx], spec, be)
    return idx, res
