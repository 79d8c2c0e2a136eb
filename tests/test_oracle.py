"""Pins the CPU oracle (oracle/psk_oracle.c) before it is trusted as the
checker: bitwise against the reference's own golden vectors
(tests/golden/golden_ref.npz, produced by the reference headers), bitwise
against the reference shim when it is built, and against the reference tests'
known answers and properties (test_kalman_seq.cpp, test_kalman_par.cpp,
test_scan.cpp).  CPU only."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from conftest import gen, max_rel_err, scalar_model

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_ref.npz"


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _cases(golden):
    return sorted({k.split("/")[0] for k in golden.files if k.startswith("s")})


def _model(golden, key):
    from oracle.oracle import GenModel
    t = int(key.split("_t")[1])
    nx = int(key.split("_nx")[1].split("_")[0])
    ny = int(key.split("_ny")[1].split("_")[0])
    g = {k: golden[f"{key}/in/{k}"] for k in ("f", "u", "q", "h", "d", "r", "m0", "p0")}
    g.update(t=t, nx=nx, ny=ny)
    return g, GenModel(g), golden[f"{key}/in/y"]


def test_golden_generator_bitwise(port, golden):
    for key in _cases(golden):
        g, _, ys = _model(golden, key)
        seed = int(key.split("_")[0][1:])
        mine = port.gen_model(seed, g["nx"], g["ny"], g["t"])
        for k in ("f", "u", "q", "h", "d", "r", "m0", "p0"):
            assert np.array_equal(mine[k], g[k]), (key, k)
        assert np.array_equal(port.simulate_data(mine, seed + 1), ys), key


@pytest.mark.parametrize("dn", ["f64", "f32"])
def test_golden_outputs_bitwise(port, golden, dn):
    dt = np.float64 if dn == "f64" else np.float32
    for key in _cases(golden):
        _, m, ys = _model(golden, key)
        for name in ("kf_run", "rts_run", "tfs_run", "bif_run"):
            a, b = getattr(port, name)(m, ys, dt)
            assert np.array_equal(a, golden[f"{key}/{dn}/{name}/0"]), (key, name)
            assert np.array_equal(b, golden[f"{key}/{dn}/{name}/1"]), (key, name)
        for alg in range(6):
            for name in ("pkf_run", "prts_run", "ptfs_run"):
                a, b = getattr(port, name)(m, ys, alg, 4, dt)
                assert np.array_equal(a, golden[f"{key}/{dn}/{name}/alg{alg}/0"]), (key, name, alg)
                assert np.array_equal(b, golden[f"{key}/{dn}/{name}/alg{alg}/1"]), (key, name, alg)


def test_golden_elements_bitwise(port, golden):
    for key in _cases(golden):
        g, m, ys = _model(golden, key)
        nx, t = g["nx"], g["t"]
        els = np.stack([port.make_filter_element(m, ys, k) for k in range(1, t + 1)])
        assert np.array_equal(els, golden[f"{key}/f64/filter_elements"])
        combs = np.stack([port.filter_combine(nx, els[i], els[(i * 7 + 3) % t])
                          for i in range(min(t, 12))])
        assert np.array_equal(combs, golden[f"{key}/f64/filter_combine"])
        kfm, kfc = port.kf_run(m, ys)
        sels = np.stack([port.make_smoother_element(m, ys, kfm[k - 1], kfc[k - 1], k)
                         for k in range(1, t + 1)])
        assert np.array_equal(sels, golden[f"{key}/f64/smoother_elements"])
        sc = np.stack([port.smoother_combine(nx, sels[i], sels[(i * 5 + 1) % t])
                       for i in range(min(t, 12))])
        assert np.array_equal(sc, golden[f"{key}/f64/smoother_combine"])


def test_golden_int64_scans(port, golden):
    for t in list(range(1, 21)) + [64]:
        v = golden[f"int64/t{t}/in"]
        n = 1 << (t - 1).bit_length() if t > 1 else 1
        vp = np.zeros(n, dtype=np.int64)
        vp[:t] = v
        for alg in range(6):
            for rev in (0, 1):
                src = v if alg == 0 else vp
                got = port.int64_scan(src, alg, 4, bool(rev))
                assert np.array_equal(got, golden[f"int64/t{t}/alg{alg}/rev{rev}"]), (t, alg, rev)


def test_port_equals_reference_shim(port, ref):
    """Fresh random cases (not in the golden set), bitwise."""
    for seed, nx, ny, t in ((91, 4, 2, 129), (92, 2, 2, 33), (93, 5, 4, 48)):
        m, ys = gen(ref, seed, nx, ny, t)
        for dt in (np.float64, np.float32):
            for alg in range(6):
                for name in ("pkf_run", "prts_run", "ptfs_run"):
                    a = getattr(port, name)(m, ys, alg, 8, dt)
                    b = getattr(ref, name)(m, ys, alg, 8, dt)
                    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---- known answers and properties of the reference tests -------------------


def test_scalar_known_answers(port):
    """test_kalman_seq.cpp:63-98 and test_kalman_par.cpp:72-93."""
    m = scalar_model(2)
    ys = np.ones((2, 1))
    mean, cov = port.kf_run(m, ys)
    np.testing.assert_allclose(mean[:, 0], [2 / 3, 7 / 8])
    np.testing.assert_allclose(cov[:, 0, 0], [2 / 3, 5 / 8])
    mean, cov = port.rts_run(m, ys)
    np.testing.assert_allclose([mean[0, 0], cov[0, 0, 0]], [3 / 4, 1 / 2])
    eta, jm = port.bif_run(m, ys)
    np.testing.assert_allclose([eta[0, 0], jm[0, 0, 0]], [1 / 2, 1 / 2])
    e1 = port.make_filter_element(m, ys, 1)  # (A,b,C,eta,J) = (0,2/3,2/3,1/3,1/3)
    np.testing.assert_allclose(e1, [0, 2 / 3, 2 / 3, 1 / 3, 1 / 3])
    e2 = port.make_filter_element(m, np.zeros((2, 1)), 2)  # (0.5, 0, 0.5, 0, 0.5)
    np.testing.assert_allclose(e2, [0.5, 0, 0.5, 0, 0.5])


def test_zero_h_reduces_to_dynamics(port):
    """test_kalman_par.cpp:95-105."""
    from oracle.oracle import GenModel
    g = port.gen_model(5, 3, 2, 4)
    g["h"][2] = 0
    m = GenModel(g)
    e = port.make_filter_element(m, np.zeros((4, 2)), 3)
    nx = 3
    assert np.abs(e[:9] - g["f"][2].ravel()).max() < 1e-14
    assert np.abs(e[9:12] - g["u"][2]).max() < 1e-14
    assert np.abs(e[12:21] - g["q"][2].ravel()).max() < 1e-14
    assert np.all(e[21:] == 0)
    assert nx == 3


def test_associativity_and_identities(port):
    """test_kalman_par.cpp:107-144."""
    from oracle.oracle import GenModel
    from oracle.oracle import Oracle  # noqa: F401
    g = port.gen_model(17, 3, 2, 16)
    ys = port.simulate_data(g, 18)
    m = GenModel(g)
    pool = [port.make_filter_element(m, ys, k) for k in range(1, 17)]
    mix = port.lib.pso_splitmix64
    import ctypes
    mix.restype = ctypes.c_uint64
    mix.argtypes = [ctypes.c_uint64]
    for trial in range(100):
        a, b, c = (pool[mix(trial * 3 + i) % 16] for i in range(3))
        lhs = port.filter_combine(3, port.filter_combine(3, a, b), c)
        rhs = port.filter_combine(3, a, port.filter_combine(3, b, c))
        assert np.abs(lhs - rhs).max() < 1e-8
    ident = np.zeros_like(pool[0])
    ident[[0, 4, 8]] = 1.0
    for e in pool[:8]:
        assert np.abs(port.filter_combine(3, ident, e) - e).max() < 1e-12
        assert np.abs(port.filter_combine(3, e, ident) - e).max() < 1e-12


def test_rts_equals_tfs_20_seeds(port):
    """test_kalman_seq.cpp:100-108."""
    for seed in range(20):
        m, ys = gen(port, seed, 4, 2, 30)
        r = port.rts_run(m, ys)
        t = port.tfs_run(m, ys)
        assert max_rel_err(t[0], t[1], *r) < 1e-9


def test_scan_work_counts(port):
    """count_work_and_span closed forms (test_scan.cpp:130-145,
    test_acceptance.cpp work_identities)."""
    for e in range(1, 11):
        t = 1 << e
        v = np.arange(1, t + 1)
        port.int64_scan(v, 1)
        assert port.lib.pso_last_scan_work() == t * e - t + 1
        port.int64_scan(v, 2)
        bl_span = port.lib.pso_last_scan_span()
        assert port.lib.pso_last_scan_work() == 3 * t - 2
        port.int64_scan(v, 3)
        assert port.lib.pso_last_scan_work() == 2 * t - 2 - e
        if t >= 4:
            assert port.lib.pso_last_scan_span() == bl_span - 2


@pytest.mark.parametrize("alg", range(6))
def test_int64_scans_match_cumsum(port, alg):
    rng = np.random.default_rng(alg)
    for t in list(range(1, 65)) + [1000]:
        v = rng.integers(-1000, 1001, t)
        n = t if alg == 0 else 1 << (t - 1).bit_length()
        vp = np.zeros(n, dtype=np.int64)
        vp[:t] = v
        got = port.int64_scan(vp, alg, 4)
        assert np.array_equal(got[:t], np.cumsum(v)), (alg, t)
        got = port.int64_scan(vp, alg, 4, reverse=True)
        assert np.array_equal(got[n - t:] if alg else got, np.cumsum(vp[::-1])[::-1][n - t:] if alg else np.cumsum(v[::-1])[::-1])


def test_contracts(port):
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        port.int64_scan(np.zeros(0), 3)          # empty
    with pytest.raises(OracleError):
        port.int64_scan(np.zeros(6), 3)          # non power of two
    with pytest.raises(OracleError):
        port.int64_scan(np.zeros(8), 5, 3)       # SenguptaB N not pow2
    port.int64_scan(np.zeros(6), 0)              # Sequential accepts any length
