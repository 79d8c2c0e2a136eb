"""The C++ drop-in end to end: a reference user's program (the unmodified
reference headers + include/parascan_b200/cuda_backend.hpp, built by
oracle/Makefile into oracle/_ref/dropin_check) runs prts_run / pkf_run /
ptfs_run with PoolBackend and with CudaBackend -- only the backend object
changes -- and every GPU result must match the reference's own result within
1e-9 (exact mode: bitwise), with the reference's exception types on errors."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "dropin_check"


def test_cpp_dropin_matches_reference(gpu):
    if not BIN.exists():
        pytest.skip("oracle/_ref/dropin_check not built (needs the reference headers)")
    p = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "DROPIN OK" in p.stdout


PSK_BENCH = ROOT / "tools" / "_bin" / "psk_bench"


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_psk_bench_verify_all_algs(gpu, precision):
    """The reference's `bench verify` grid (gen_model inputs, f64 sequential
    oracle, the reference's gating tolerances bench.hpp rel_err_tolerance)
    with the CUDA backend: every method x every ScanAlg (+ DLB) passes."""
    if not PSK_BENCH.exists():
        pytest.skip("tools/_bin/psk_bench not built (needs the reference headers)")
    p = subprocess.run([str(PSK_BENCH), "verify", "--T", "64", "1000", "4096", "--methods", "pkf",
                        "prts", "ptfs", "--algs", "all", "--precision", precision],
                       capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:])
    assert p.returncode == 0, p.stdout + p.stderr
    rows = [r.split(",") for r in p.stdout.strip().splitlines()[1:]]
    assert len(rows) == 3 * 3 * 7
    bar = 1e-9 if precision == "f64" else 1e-2
    for r in rows:
        assert r[4] == "max_rel_err" and float(r[5]) <= bar, r


def test_psk_bench_run_rows(gpu, tmp_path):
    """`run` emits the reference's CSV schema with the GPU metrics."""
    if not PSK_BENCH.exists():
        pytest.skip("tools/_bin/psk_bench not built")
    out = tmp_path / "r.csv"
    p = subprocess.run([str(PSK_BENCH), "run", "--T", "65536", "--methods", "prts", "--runs", "3",
                        "--warmup", "1", "--model", "cv", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "method,alg,T,precision,metric,value,seed,threads,devices"
    metrics = {r.split(",")[4]: float(r.split(",")[5]) for r in lines[1:]}
    for k in ("max_rel_err", "wall_median_s", "steps_per_s", "device_median_s",
              "device_steps_per_s", "hbm_frac", "fp_frac"):
        assert k in metrics, k
    assert metrics["max_rel_err"] < 1e-9
    assert 0 < metrics["device_median_s"] < metrics["wall_median_s"]
