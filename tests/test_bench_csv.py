"""tools/_bin/psk_bench (the reference's benchmark workbench on the CUDA
backend, tools/psk_bench.cpp) without a GPU: argument errors exit 2 like the
reference CLI, and `--backend pool` produces the reference's own CSV rows
(schema bench.hpp:108-188) -- the same program the GPU rows come from."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tools" / "_bin" / "psk_bench"

pytestmark = pytest.mark.skipif(not BIN.exists(), reason="tools/_bin/psk_bench not built")


def test_bad_arguments_exit_2():
    for args in (["bogus"], ["run", "--nx", "17"], ["run", "--runs", "2", "--warmup", "2"],
                 ["run", "--devices", "3"], ["run", "--backend", "pool", "--algs",
                                             "decoupled_lookback"]):
        p = subprocess.run([str(BIN), *args], capture_output=True, text=True, timeout=60)
        assert p.returncode == 2, (args, p.stderr)


def test_pool_rows_reference_schema(tmp_path):
    out = tmp_path / "pool.csv"
    p = subprocess.run([str(BIN), "run", "--backend", "pool", "--T", "64", "256", "--methods",
                        "prts", "seq_kf", "--runs", "3", "--warmup", "1", "--threads", "2",
                        "--out", str(out)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "method,alg,T,precision,metric,value,seed,threads,devices"
    rows = [ln.split(",") for ln in lines[1:]]
    assert all(len(r) == 9 for r in rows)
    # deterministic order (bench.hpp sort_rows): method, alg, T, metric
    keys = [(r[0], r[1], int(r[2]), r[4]) for r in rows]
    assert keys == sorted(keys)
    err = {(r[0], int(r[2])): float(r[5]) for r in rows if r[4] == "max_rel_err"}
    assert err[("seq_kf", 64)] == 0.0 and err[("prts", 256)] < 1e-9


def test_cuda_backend_fails_loudly_without_device():
    p = subprocess.run([str(BIN), "run", "--T", "64", "--methods", "prts"], capture_output=True,
                       text=True, timeout=60)
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert p.returncode == 2 and "no CUDA device" in p.stderr
