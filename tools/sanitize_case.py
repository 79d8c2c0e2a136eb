"""Small PKF / PRTS / PTFS runs over every ScanAlg (fast + wide path), for
compute-sanitizer (tests/test_gpu_sanitizer.py)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200.synthetic import cv_model

    m, ys = cv_model(3000, seed=1)
    for chunk in (0, 3):
        be = psk.CudaBackend(0, chunk=chunk)
        for alg in range(7):
            spec = psk.ScanSpec(psk.ScanAlg(alg), 4)
            psk.pkf_run(m, ys, spec, be)
            psk.prts_run(m, ys, spec, be)
            psk.ptfs_run(m, ys, spec, be)
    # wide path (nx = 6, ny = 3)
    rng = np.random.default_rng(0)
    nx, ny, t = 6, 3, 300
    q_, _ = np.linalg.qr(rng.standard_normal((nx, nx)))
    F = np.broadcast_to(0.9 * q_, (t, nx, nx)).copy()
    Q = np.broadcast_to(np.eye(nx) * 0.1, (t, nx, nx)).copy()
    H = np.broadcast_to(rng.standard_normal((ny, nx)), (t, ny, nx)).copy()
    R = np.broadcast_to(np.eye(ny), (t, ny, ny)).copy()
    mw = psk.Lgssm(f=F, u=np.zeros((t, nx)), q=Q, h=H, d=np.zeros((t, ny)), r=R,
                   prior_mean=np.zeros(nx), prior_cov=np.eye(nx), t=t)
    yw = rng.standard_normal((t, ny))
    be = psk.CudaBackend(0)
    for alg in (3, 6):
        psk.prts_run(mw, yw, psk.ScanSpec(psk.ScanAlg(alg)), be)
    print("sanitize case done")


if __name__ == "__main__":
    main()
