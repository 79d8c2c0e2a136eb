"""Edge semantics of the fast path's arithmetic and of the Python API.

* The branch-free reciprocal / reciprocal square root (psk_mat.cuh srcp /
  srsqrt) that replace IEEE division in the fast kernels must give the IEEE
  result the reference computes (mat.hpp divides in IEEE) within 2 ulp --
  including subnormal pivots, where an FTZ seed would flush to zero and yield
  inf, and huge arguments whose reciprocal is subnormal.
* Device-space calls made without an explicit stream are ordered after the
  work torch queued on its current stream (inputs produced by torch
  just before the call must be complete when the kernels read them).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import ROOT, max_rel_err

pytestmark = pytest.mark.gpu

TOOLS = ROOT / "paper_2511_10363_b200" / "lib" / "libpsk_tools.so"


_RCP_CHILD = """
import ctypes as C, sys
import numpy as np
x = np.load(sys.argv[2])
lib = C.CDLL(sys.argv[1])
r = np.empty_like(x)
q = np.empty_like(x)
st = lib.psk_tool_rcp(int(x.dtype == np.float64), C.c_void_p(x.ctypes.data),
                      C.c_void_p(r.ctypes.data), C.c_void_p(q.ctypes.data), int(x.size))
np.savez(sys.argv[3], r=r, q=q, st=st)
"""


def _rcp(x: np.ndarray, tmp):
    """srcp / srsqrt on the device.  The measurement-tool library carries its
    own static CUDA runtime, so it runs in a child process rather than next to
    libpsk.so and torch in the test process."""
    import subprocess
    import sys
    np.save(tmp / "x.npy", x)
    subprocess.run([sys.executable, "-c", _RCP_CHILD, str(TOOLS), str(tmp / "x.npy"),
                    str(tmp / "out.npz")], check=True, timeout=300)
    d = np.load(tmp / "out.npz")
    assert int(d["st"]) == 0
    return d["r"], d["q"]


def _ulps(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Distance in units in the last place (finite same-sign values)."""
    it = np.int64 if a.dtype == np.float64 else np.int32
    return np.abs(a.view(it).astype(np.int64) - b.view(it).astype(np.int64))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_reciprocals_match_ieee_incl_subnormal(gpu, dtype, tmp_path):
    fi = np.finfo(dtype)
    rng = np.random.default_rng(0)
    normal = rng.uniform(0.5, 2.0, 200) * 2.0 ** rng.integers(-60, 60, 200)
    tiny = [fi.tiny, fi.tiny / 3, fi.tiny * 0.9, fi.smallest_subnormal * 2 ** 20,
            fi.smallest_subnormal * 2 ** 40 if dtype == np.float64 else fi.tiny / 8]
    huge = [fi.max / 2, fi.max / 7, float(fi.max) ** 0.5 * 3, 2.0 ** (fi.maxexp - 3)]
    x = np.array(list(normal) + tiny + huge, dtype=dtype)
    x = np.concatenate([x, -x[: len(normal) // 2]])
    with np.errstate(over="ignore", divide="ignore"):
        want_r = (dtype(1) / x).astype(dtype)
        pos = x > 0
        want_q = (dtype(1) / np.sqrt(x[pos])).astype(dtype)
    got_r, got_q = _rcp(x, tmp_path)
    fin = np.isfinite(want_r) & (want_r != 0)
    assert np.all(np.isfinite(got_r[fin])), "a finite IEEE reciprocal became inf/0"
    assert _ulps(got_r[fin], want_r[fin]).max() <= 2
    assert np.all(np.isfinite(got_q[pos]))
    assert _ulps(got_q[pos], want_q).max() <= 2


def test_device_inputs_ordered_after_torch_stream(gpu):
    """Inputs written by torch right before the call (no explicit stream on
    the backend, no synchronisation) are the ones the kernels read."""
    import torch

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model

    m, ys = cv_model(1 << 16, seed=5)
    dev = torch.device("cuda", gpu)
    be = psk.CudaBackend(gpu, chunk=0)
    want = psk.prts_run(m, ys, psk.ScanSpec(psk.ScanAlg.DecoupledLookback, 1), be)
    for trial in range(3):
        yd = torch.zeros((m.t, 2), dtype=torch.float64, device=dev)
        big = torch.randn(4096, 4096, device=dev, dtype=torch.float64)
        for _ in range(4):  # keep torch's stream busy before the input lands
            big = big @ big * 1e-3
        yd.copy_(torch.as_tensor(ys), non_blocking=False)
        yd += big[0, 0] * 0  # last writer of yd is a kernel queued on torch's stream
        md = psk.Lgssm(**{k: torch.as_tensor(getattr(m, k), device=dev)
                          for k in ("f", "u", "q", "h", "d", "r", "prior_mean",
                                    "prior_cov")}, t=m.t)
        out = psk.prts_run(md, yd, psk.ScanSpec(psk.ScanAlg.DecoupledLookback, 1), be)
        got_m = out.mean.cpu().numpy()
        got_c = out.cov.cpu().numpy()
        assert max_rel_err(got_m, got_c, want.mean, want.cov) == 0.0, trial


def test_out_buffer_checks(gpu):
    import torch

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model

    m, ys = cv_model(64, seed=1)
    be = psk.CudaBackend(gpu)
    spec = psk.ScanSpec(psk.ScanAlg.InplaceLaFi, 1)
    ok = psk.GaussianStats(np.empty((64, 4)), np.empty((64, 4, 4)))
    psk.prts_run(m, ys, spec, be, out=ok)
    bad = [
        psk.GaussianStats(np.empty((64, 4), np.float32), np.empty((64, 4, 4))),
        psk.GaussianStats(np.empty((64, 8))[:, ::2], np.empty((64, 4, 4))),
        psk.GaussianStats(torch.empty(64, 4, dtype=torch.float64), np.empty((64, 4, 4))),
    ]
    for o in bad:
        with pytest.raises((ValueError, psk.DimensionMismatch)):
            psk.prts_run(m, ys, spec, be, out=o)
    dev = torch.device("cuda", gpu)
    md = psk.Lgssm(**{k: torch.as_tensor(getattr(m, k), device=dev)
                      for k in ("f", "u", "q", "h", "d", "r", "prior_mean", "prior_cov")},
                   t=m.t)
    yd = torch.as_tensor(ys, device=dev)
    with pytest.raises(ValueError):  # host outputs for a device-space model
        psk.prts_run(md, yd, spec, be, out=psk.GaussianStats(
            torch.empty(64, 4, dtype=torch.float64), torch.empty(64, 4, 4, dtype=torch.float64)))
