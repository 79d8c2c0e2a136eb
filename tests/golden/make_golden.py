"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference headers through oracle/_ref/libparascan_ref.so
(built by `make -C oracle` from /root/reference) and stores inputs and outputs
as compressed npz.  The files are committed; the GPU box (which has no
/root/reference) checks the oracle restatement and the CUDA path against them.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle.oracle import GenModel, Oracle  # noqa: E402

CASES = [  # (seed, nx, ny, T): shapes of the reference tests
    (3, 4, 2, 37),    # ragged T (padding to 64)
    (10, 4, 2, 64),   # power of two (test_kalman_par.cpp:163-191 sizes)
    (40, 4, 2, 60),   # ptfs test sizes (test_kalman_par.cpp:209-227)
    (5, 3, 2, 20),
    (17, 1, 1, 9),
    (8, 6, 3, 16),
]
ALGS = range(6)


def main() -> None:
    ref = Oracle("ref")
    out: dict[str, np.ndarray] = {}
    for seed, nx, ny, t in CASES:
        key = f"s{seed}_nx{nx}_ny{ny}_t{t}"
        g = ref.gen_model(seed, nx, ny, t)
        ys = ref.simulate_data(g, seed + 1)
        m = GenModel(g)
        for k in ("f", "u", "q", "h", "d", "r", "m0", "p0"):
            out[f"{key}/in/{k}"] = g[k]
        out[f"{key}/in/y"] = ys
        for dt, dn in ((np.float64, "f64"), (np.float32, "f32")):
            for name in ("kf_run", "rts_run", "tfs_run", "bif_run"):
                a, b = getattr(ref, name)(m, ys, dt)
                out[f"{key}/{dn}/{name}/0"] = a
                out[f"{key}/{dn}/{name}/1"] = b
            for alg in ALGS:
                for name in ("pkf_run", "prts_run", "ptfs_run"):
                    a, b = getattr(ref, name)(m, ys, alg, 4, dt)
                    out[f"{key}/{dn}/{name}/alg{alg}/0"] = a
                    out[f"{key}/{dn}/{name}/alg{alg}/1"] = b
        # elements and operators (kalman_elems.hpp)
        els = np.stack([ref.make_filter_element(m, ys, k) for k in range(1, t + 1)])
        out[f"{key}/f64/filter_elements"] = els
        combs = np.stack([ref.filter_combine(nx, els[i], els[(i * 7 + 3) % t])
                          for i in range(min(t, 12))])
        out[f"{key}/f64/filter_combine"] = combs
        kfm, kfc = ref.kf_run(m, ys)
        sels = np.stack([ref.make_smoother_element(m, ys, kfm[k - 1], kfc[k - 1], k)
                         for k in range(1, t + 1)])
        out[f"{key}/f64/smoother_elements"] = sels
        out[f"{key}/f64/smoother_combine"] = np.stack(
            [ref.smoother_combine(nx, sels[i], sels[(i * 5 + 1) % t]) for i in range(min(t, 12))])
    # Int64Elems scans (test_scan.cpp:45-67 shape): every alg, T = 1..20, 64
    for t in list(range(1, 21)) + [64]:
        v = (np.arange(t, dtype=np.int64) * 37 % 2001) - 1000
        n = 1 << (t - 1).bit_length() if t > 1 else 1
        vp = np.zeros(n, dtype=np.int64)
        vp[:t] = v
        out[f"int64/t{t}/in"] = v
        for alg in ALGS:
            for rev in (0, 1):
                src = v if alg == 0 else vp
                out[f"int64/t{t}/alg{alg}/rev{rev}"] = ref.int64_scan(src, alg, 4, bool(rev))
    np.savez_compressed(HERE / "golden_ref.npz", **out)
    print(f"wrote {len(out)} arrays to {HERE / 'golden_ref.npz'}")


if __name__ == "__main__":
    main()
