"""CUDA shard phases (psk_shard_* / psk_fold_*) on one GPU with G virtual
ranks (NCCL forbids two ranks on one GPU): the time-sharded PRTS must match the
sequential oracle at 1e-9 (FP64) for several G, chunk lengths and scan
algorithms, with uneven shards."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import gen, max_rel_err

pytestmark = pytest.mark.gpu


def _virtual_sharded_prts(psk, m, ys, G, chunk, alg, gpu):
    import torch

    from paper_2511_10363_b200.distributed import CudaShardEngine, shard_flags, shard_range
    T = m.t
    tt = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    engines, spans = [], []
    for g in range(G):
        lo, hi = shard_range(T, g, G)
        hi_in = min(hi + 1, T)
        s_in = slice(lo, hi_in)
        mg = psk.Lgssm(f=tt(m.f[s_in]), u=tt(m.u[s_in]), q=tt(m.q[s_in]), h=tt(m.h[s_in]),
                       d=tt(m.d[s_in]), r=tt(m.r[s_in]), prior_mean=tt(m.prior_mean),
                       prior_cov=tt(m.prior_cov), t=hi_in - lo)
        be = psk.CudaBackend(gpu, mode="fast", chunk=chunk)
        engines.append(CudaShardEngine(be, mg, tt(ys[s_in]), shard_flags(g, G), hi - lo))
        spans.append((lo, hi))
    spec = psk.ScanSpec(psk.ScanAlg(alg), 4)
    a = [e.filter_reduce(spec) for e in engines]
    stats = []
    for g, e in enumerate(engines):
        carry = e.fold("filter", a[:g]) if g > 0 else None
        mean, cov = e.stats(spans[g][1] - spans[g][0])
        e.filter_finish(carry, mean, cov)
        stats.append((mean, cov))
    s = [e.smoother_reduce(spec, *stats[g]) for g, e in enumerate(engines)]
    for g, e in enumerate(engines):
        carry = e.fold("smoother", s[g + 1:]) if g < G - 1 else None
        e.smoother_finish(carry, *stats[g])
    mean = np.concatenate([st[0].cpu().numpy() for st in stats])
    cov = np.concatenate([st[1].cpu().numpy() for st in stats])
    return mean, cov


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("alg,chunk", [(6, 8), (3, 4), (2, 1)])
def test_virtual_sharded_prts(gpu, port, G, alg, chunk):
    import paper_2511_10363_b200 as psk
    m, ys = gen(port, 30 + G, 4, 2, 999)
    rts = port.rts_run(m, ys)
    mean, cov = _virtual_sharded_prts(psk, m, ys, G, chunk, alg, gpu)
    assert max_rel_err(mean, cov, *rts) < 1e-9


def test_virtual_sharded_tracking_large(gpu, port):
    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model
    m, ys = cv_model(1 << 18, seed=4)
    rts = port.rts_run(m, ys)
    mean, cov = _virtual_sharded_prts(psk, m, ys, 8, 32, 6, gpu)
    assert max_rel_err(mean, cov, *rts) < 1e-9


def test_shard_requires_device_inputs(gpu, port):
    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.distributed import CudaShardEngine
    m, ys = gen(port, 1, 4, 2, 10)
    be = psk.CudaBackend(gpu)
    with pytest.raises(ValueError):
        CudaShardEngine(be, m, ys, 3, 10)


def _virtual_sharded_ptfs(psk, m, ys, h, chunk, alg, gpu):
    """The sharded PTFS (distributed.ptfs_sharded) with 2h virtual ranks on one
    GPU: h forward shard engines (PSK_SHARD_FILTERED) and h backward ones over
    the same step ranges; the exchanges done in-process."""
    import torch

    from paper_2511_10363_b200 import _lib
    from paper_2511_10363_b200.distributed import (CudaShardEngine, shard_flags, shard_model,
                                                   shard_range)
    T = m.t
    dev = torch.device("cuda", gpu)
    spec = psk.ScanSpec(psk.ScanAlg(alg), 4)
    fwd, bwd, spans = [], [], []
    for i in range(h):
        lo, hi = shard_range(T, i, h)
        ms, yss = shard_model(m, ys, lo, hi, device=dev)
        f = shard_flags(i, h)
        fwd.append(CudaShardEngine(psk.CudaBackend(gpu, chunk=chunk), ms, yss,
                                   f | _lib.PSK_SHARD_FILTERED, hi - lo))
        bwd.append(CudaShardEngine(psk.CudaBackend(gpu, chunk=chunk), ms, yss, f, hi - lo))
        spans.append((lo, hi))
    a = [e.filter_reduce(spec) for e in fwd]
    s = [e.backward_reduce(spec) for e in bwd]
    out = []
    for i in range(h):
        t = spans[i][1] - spans[i][0]
        fm, fc = fwd[i].stats(t)
        fwd[i].filter_finish(fwd[i].fold("filter", a[:i]) if i > 0 else None, fm, fc)
        carry = bwd[i].fold("backward", s[i + 1:]) if i < h - 1 else None
        mean, cov = bwd[i].stats(t)
        bwd[i].backward_finish(carry, fm, fc, mean, cov)
        out.append((mean.cpu().numpy(), cov.cpu().numpy()))
    return np.concatenate([o[0] for o in out]), np.concatenate([o[1] for o in out])


@pytest.mark.parametrize("h", [1, 2, 4])
@pytest.mark.parametrize("alg,chunk", [(6, 8), (3, 4), (2, 1)])
def test_virtual_sharded_ptfs_halves(gpu, port, h, alg, chunk):
    """PTFS on disjoint halves of 2h virtual ranks (each half time-sharded in
    h shards) matches the sequential RTS oracle, like the one-context PTFS
    (test_kalman_par.cpp:209-227: ptfs == rts at 1e-9)."""
    import paper_2511_10363_b200 as psk
    m, ys = gen(port, 40 + h, 4, 2, 777)
    rts = port.rts_run(m, ys)
    mean, cov = _virtual_sharded_ptfs(psk, m, ys, h, chunk, alg, gpu)
    assert max_rel_err(mean, cov, *rts) < 1e-9
    one = psk.ptfs_run(m, ys, psk.ScanSpec(psk.ScanAlg(alg), 4),
                       psk.CudaBackend(gpu, chunk=chunk))
    assert max_rel_err(mean, cov, one.mean, one.cov) < 1e-12


def test_virtual_sharded_ptfs_tracking_large(gpu, port):
    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model
    m, ys = cv_model(1 << 18, seed=6)
    rts = port.rts_run(m, ys)
    mean, cov = _virtual_sharded_ptfs(psk, m, ys, 4, 32, 6, gpu)
    assert max_rel_err(mean, cov, *rts) < 1e-9


@pytest.mark.parametrize("devs", [[0, 0], [0, 0, 0], [0, 0, 0, 0], [0] * 8])
def test_multi_device_context(gpu, port, devs):
    """psk_create_multi: one process driving several members (streams of the
    one GPU here; separate GPUs over NVLink on a multi-GPU box): PKF / PRTS
    time-sharded over the members, PTFS on the two halves, host and device
    inputs, against the sequential oracle (1e-9)."""
    import torch

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model
    m, ys = gen(port, 50 + len(devs), 4, 2, 3001)
    kf = port.kf_run(m, ys)
    rts = port.rts_run(m, ys)
    be = psk.CudaBackend(devs)
    for alg in (6, 3):
        spec = psk.ScanSpec(psk.ScanAlg(alg), 16)
        got = psk.prts_run(m, ys, spec, be)
        assert max_rel_err(got.mean, got.cov, *rts) < 1e-9, ("prts", alg)
        got = psk.pkf_run(m, ys, spec, be)
        assert max_rel_err(got.mean, got.cov, *kf) < 1e-9, ("pkf", alg)
        got = psk.ptfs_run(m, ys, spec, be, be, len(devs))
        assert max_rel_err(got.mean, got.cov, *rts) < 1e-9, ("ptfs", alg)
    assert be.last_launch_count() > 0
    # device-space inputs and outputs
    dev = torch.device("cuda", gpu)
    mc, yc = cv_model(1 << 16, seed=9)
    want = port.rts_run(mc, yc)
    md = psk.Lgssm(**{k: torch.as_tensor(getattr(mc, k), device=dev)
                      for k in ("f", "u", "q", "h", "d", "r", "prior_mean", "prior_cov")},
                   t=mc.t)
    got = psk.prts_run(md, torch.as_tensor(yc, device=dev),
                       psk.ScanSpec(psk.ScanAlg.DecoupledLookback), be)
    assert max_rel_err(got.mean.cpu(), got.cov.cpu(), *want) < 1e-9


def test_multi_device_batch_and_fallbacks(gpu, port):
    """Batches on a multi-device context are split between the members; dims
    without shard phases (nx > 4) and tiny series run on the first member."""
    import paper_2511_10363_b200 as psk
    be = psk.CudaBackend([0, 0])
    series = [gen(port, 60 + i, 4, 2, 500 + 37 * i) for i in range(5)]
    outs = psk.prts_run_batch([s[0] for s in series], [s[1] for s in series],
                              psk.ScanSpec(psk.ScanAlg.DecoupledLookback), be)
    for (m, ys), o in zip(series, outs):
        assert max_rel_err(o.mean, o.cov, *port.rts_run(m, ys)) < 1e-9
    m, ys = gen(port, 70, 8, 4, 300)
    got = psk.prts_run(m, ys, psk.ScanSpec(psk.ScanAlg.InplaceLaFi), be)
    assert max_rel_err(got.mean, got.cov, *port.rts_run(m, ys)) < 1e-9
    m, ys = gen(port, 71, 4, 2, 1)
    got = psk.prts_run(m, ys, psk.ScanSpec(psk.ScanAlg.InplaceLaFi), be)
    assert max_rel_err(got.mean, got.cov, *port.rts_run(m, ys)) < 1e-9


def test_multi_device_f32_and_short_series(gpu, port):
    """FP32 through a multi-device context on the stationary tracking model
    (FP32 gate 1e-4 vs the f64 oracle), and series shorter than the member
    count (one member runs them)."""
    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model
    m64, ys64 = cv_model(1 << 15, seed=8)
    m32, ys32 = cv_model(1 << 15, seed=8, dtype=np.float32)
    rts = port.rts_run(m64, ys64)
    be = psk.CudaBackend([0, 0, 0, 0])
    spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback)
    got = psk.prts_run(m32, ys32, spec, be)
    assert max_rel_err(got.mean, got.cov, *rts) < 1e-4
    got = psk.ptfs_run(m32, ys32, spec, be, be, 4)
    assert max_rel_err(got.mean, got.cov, *rts) < 1e-4
    be8 = psk.CudaBackend([0] * 8)
    for t in (2, 5, 9):
        m, ys = gen(port, 80 + t, 4, 2, t)
        ref = port.rts_run(m, ys)
        got = psk.prts_run(m, ys, spec, be8)
        assert max_rel_err(got.mean, got.cov, *ref) < 1e-9, t
        got = psk.ptfs_run(m, ys, spec, be8, be8, 8)
        assert max_rel_err(got.mean, got.cov, *ref) < 1e-9, t


def test_virtual_sharded_ptfs_f32(gpu, port):
    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model
    m64, ys64 = cv_model(1 << 16, seed=12)
    m32, ys32 = cv_model(1 << 16, seed=12, dtype=np.float32)
    rts = port.rts_run(m64, ys64)
    mean, cov = _virtual_sharded_ptfs(psk, m32, ys32, 3, 0, 6, gpu)
    assert max_rel_err(mean, cov, *rts) < 1e-4
