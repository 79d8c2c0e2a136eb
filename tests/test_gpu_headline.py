"""Parity at the BASELINE.json headline configurations.

The north star's tolerance (1e-9 FP64, 1e-4 FP32 on means and covariances,
max |a-b|/(1+|b|) as bench.hpp:216-237) checked against the CPU oracle's
sequential kf_run / rts_run at the sizes the benchmark and BASELINE quote:

* configs[1] top of the sweep: PKF and PRTS at T = 2^22, FP64 and FP32,
  damped constant-velocity tracking, decoupled look-back and
  Ladner-Fischer;
* configs[2]: PTFS at T = 2^20, one context and forward || backward on two
  contexts (the reference's devices = 2 path, kalman_par.hpp:207-238);
* configs[4] on a stated subset: 4 of the 64 series -- series b is the
  reference's gen_model(s + b, 16, 8, 1) broadcast over T = 2^20 (stride-0
  fields), with y from simulate_data on that model over T steps (seed
  s + b + 1) -- through one psk_prts_batch call, FP64;
* configs[3] at its full T = 2^24 is checked by bench.py's parity leg on the
  very output it times (the "parity" object of the bench line).

Match: tests/test_kalman_par.cpp:179-191 (prts vs rts_run), bench.hpp:216-237.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import max_rel_err

pytestmark = pytest.mark.gpu

TOL64 = 1e-9
TOL32 = 1e-4


@pytest.fixture(scope="module")
def psk():
    import paper_2511_10363_b200 as p
    return p


@pytest.fixture(scope="module")
def cv22(port):
    """(model64, ys64, model32, ys32, kf, rts) at T = 2^22; the oracle's filter
    and smoother run concurrently (ctypes releases the GIL)."""
    from paper_2511_10363_b200.synthetic import cv_model
    t = 1 << 22
    m64, ys64 = cv_model(t, seed=11, time_varying=False)
    m32, ys32 = cv_model(t, seed=11, dtype=np.float32, time_varying=False)
    with ThreadPoolExecutor(2) as ex:
        kf = ex.submit(port.kf_run, m64, ys64)
        rts = ex.submit(port.rts_run, m64, ys64)
        return m64, ys64, m32, ys32, kf.result(), rts.result()


def _per_step(psk, m, dtype):
    """The same model written per step (the reference API's layout)."""
    t = int(m.t)

    def ps(a):
        a = np.asarray(a, dtype=dtype)
        return np.ascontiguousarray(np.broadcast_to(a, (t, *a.shape)))

    return psk.Lgssm(f=ps(m.f), u=ps(m.u), q=ps(m.q), h=ps(m.h), d=ps(m.d), r=ps(m.r),
                     prior_mean=np.asarray(m.prior_mean, dtype), prior_cov=np.asarray(
                         m.prior_cov, dtype), t=t)


@pytest.mark.parametrize("alg", [6, 3])
def test_prts_pkf_2p22_f64(psk, gpu, cv22, alg):
    m64, ys64, _, _, kf, rts = cv22
    be = psk.CudaBackend(gpu)
    mp = _per_step(psk, m64, np.float64)  # per-step (time-varying) layout
    spec = psk.ScanSpec(psk.ScanAlg(alg), 16)
    got = psk.prts_run(mp, ys64, spec, be)
    e = max_rel_err(got.mean, got.cov, *rts)
    assert e < TOL64, e
    got = psk.pkf_run(m64, ys64, spec, be)  # broadcast layout
    e = max_rel_err(got.mean, got.cov, *kf)
    assert e < TOL64, e


def test_prts_pkf_2p22_f32(psk, gpu, cv22):
    _, _, m32, ys32, kf, rts = cv22
    be = psk.CudaBackend(gpu)
    spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback, 16)
    got = psk.prts_run(_per_step(psk, m32, np.float32), ys32, spec, be)
    e = max_rel_err(got.mean, got.cov, *rts)
    assert e < TOL32, e
    got = psk.pkf_run(m32, ys32, spec, be)
    e = max_rel_err(got.mean, got.cov, *kf)
    assert e < TOL32, e


def test_ptfs_2p20_one_and_two_contexts(psk, gpu, port):
    """configs[2]: PTFS at T = 2^20 vs rts_run; forward || backward on two
    contexts gives the one-context result bitwise (test_kalman_par.cpp:209-227)."""
    from paper_2511_10363_b200.synthetic import cv_model
    m, ys = cv_model(1 << 20, seed=13)
    rts = port.rts_run(m, ys)
    fwd, bwd = psk.CudaBackend(gpu), psk.CudaBackend(gpu)
    spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback, 16)
    one = psk.ptfs_run(m, ys, spec, fwd)
    e = max_rel_err(one.mean, one.cov, *rts)
    assert e < TOL64, e
    two = psk.ptfs_run(m, ys, spec, fwd, bwd, 2)
    assert np.array_equal(one.mean, two.mean) and np.array_equal(one.cov, two.cov)
    lafi = psk.ptfs_run(m, ys, psk.ScanSpec(psk.ScanAlg.InplaceLaFi, 16), fwd, bwd, 2)
    e = max_rel_err(lafi.mean, lafi.cov, *rts)
    assert e < TOL64, e


def _config5_series(port, psk, b: int, t: int, seed: int = 0):
    """Series b of BASELINE configs[4]: the time-
    invariant model gen_model(seed + b, 16, 8, 1) broadcast over t steps and
    y = simulate_data(that model over t steps, seed + b + 1)."""
    g = port.gen_model(seed + b, 16, 8, 1)
    blk = {k: g[k][0] for k in ("f", "u", "q", "h", "d", "r")}
    gt = dict(blk, m0=g["m0"], p0=g["p0"], t=t, nx=16, ny=8, bcast=0x3F)
    ys = port.simulate_data(gt, seed + b + 1)
    m = psk.Lgssm(**blk, prior_mean=g["m0"], prior_cov=g["p0"], t=t)
    return m, ys


def test_config5_subset_2p20_f64(psk, gpu, port):
    """configs[4] on a stated subset: series 0, 21, 42, 63 of the 64."""
    t = 1 << 20
    picks = (0, 21, 42, 63)
    series = [_config5_series(port, psk, b, t) for b in picks]
    with ThreadPoolExecutor(len(series)) as ex:
        refs = list(ex.map(lambda s: port.rts_run(*s), series))
    be = psk.CudaBackend(gpu)
    outs = psk.prts_run_batch([s[0] for s in series], [s[1] for s in series],
                              psk.ScanSpec(psk.ScanAlg.DecoupledLookback), be)
    for b, o, r in zip(picks, outs, refs):
        e = max_rel_err(o.mean, o.cov, *r)
        assert e < TOL64, (b, e)


def test_config5_ptfs_and_pkf_tiled(psk, gpu, port):
    """The two-filter smoother and the filter at nx = 16, ny = 8 through the
    register-tiled kernels (PTFS backward pass fused with the two-filter
    combination), one configs[4] series at T = 2^17, vs the sequential
    oracle; the runtime-dimension kernels (option "tile" = 0) agree."""
    t = 1 << 17
    m, ys = _config5_series(port, psk, 5, t)
    with ThreadPoolExecutor(2) as ex:
        rts = ex.submit(port.rts_run, m, ys)
        kf = ex.submit(port.kf_run, m, ys)
        rts, kf = rts.result(), kf.result()
    be = psk.CudaBackend(gpu)
    spec = psk.ScanSpec(psk.ScanAlg.DecoupledLookback)
    be.set_profile(True)
    got = psk.ptfs_run(m, ys, spec, be)
    assert any(n == "tile_bwd_finish_tf_combine" for n, _ in be.last_profile())
    e = max_rel_err(got.mean, got.cov, *rts)
    assert e < TOL64, e
    got = psk.pkf_run(m, ys, spec, be)
    e = max_rel_err(got.mean, got.cov, *kf)
    assert e < TOL64, e
    wide = psk.CudaBackend(gpu)
    wide.set_option("tile", 0)
    w = psk.prts_run(m, ys, spec, wide)
    got = psk.prts_run(m, ys, spec, be)
    assert max_rel_err(got.mean, got.cov, w.mean, w.cov) < 1e-10
