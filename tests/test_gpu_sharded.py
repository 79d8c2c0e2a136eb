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
