"""Shared fixtures.  GPU tests are marked @pytest.mark.gpu and call the CUDA
path through the C-ABI (libpsk.so); everything else runs on CPU."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_LIB, Oracle
    if not REF_LIB.exists():
        pytest.skip("oracle/_ref not built")
    return Oracle("ref")


def gen(orc, seed, nx, ny, t):
    """gen_model/simulate_data with the reference seed convention (data seed
    = model seed + 1, bench.hpp:266-267) -> (Lgssm, ys)."""
    from paper_2511_10363_b200.api import Lgssm
    g = orc.gen_model(seed, nx, ny, t)
    ys = orc.simulate_data(g, seed + 1)
    m = Lgssm(f=g["f"], u=g["u"], q=g["q"], h=g["h"], d=g["d"], r=g["r"],
              prior_mean=g["m0"], prior_cov=g["p0"], t=t)
    return m, ys


def scalar_model(t):
    """F=Q=H=R=1, zero offsets, prior (0, 1) (test_kalman_par.cpp:14-30)."""
    from paper_2511_10363_b200.api import Lgssm
    one = np.ones((t, 1, 1))
    z = np.zeros((t, 1))
    return Lgssm(f=one.copy(), u=z.copy(), q=one.copy(), h=one.copy(), d=z.copy(),
                 r=one.copy(), prior_mean=np.zeros(1), prior_cov=np.eye(1), t=t)


def max_rel_err(got_mean, got_cov, ref_mean, ref_cov):
    """max |a-b|/(1+|b|) over means and covariances (test_util.hpp:88-102,
    bench.hpp:216-237)."""
    gm = np.asarray(got_mean.cpu() if hasattr(got_mean, "cpu") else got_mean, dtype=np.float64)
    gc = np.asarray(got_cov.cpu() if hasattr(got_cov, "cpu") else got_cov, dtype=np.float64)
    e1 = np.max(np.abs(gm - ref_mean) / (1 + np.abs(ref_mean))) if ref_mean.size else 0.0
    e2 = np.max(np.abs(gc - ref_cov) / (1 + np.abs(ref_cov))) if ref_cov.size else 0.0
    return float(max(e1, e2))


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return 0
