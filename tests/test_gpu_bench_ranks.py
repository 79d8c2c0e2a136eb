"""bench.py's N > 1 path end to end on the one GPU of the test box: two
torchrun ranks (gloo instead of NCCL, both on GPU 0 -- PSK_BENCH_* test
knobs) run the time-sharded PRTS, the max-over-ranks timing, the sharded e2e
and the parity leg (oracle result broadcast, every rank checks its shard),
and rank 0 prints one JSON line with n_gpus = 2."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_two_ranks_one_gpu(gpu):
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, PSK_BENCH_DEVICE="0", PSK_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"),
           "--gpus", "2", "--log2t", "18", "--steps", "4", "--warmup", "3"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "time-sharded x2"
    assert d["parity"]["pass"] and d["parity"]["max_rel_err"] < 1e-9
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["value"] > 0 and d["gpu_launches"] > 0


def test_bench_spawn_refuses_missing_gpus(gpu):
    """--gpus N without torchrun re-launches itself, and fails loudly when
    fewer GPUs are visible."""
    import torch
    n = torch.cuda.device_count()
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n + 1),
                        "--log2t", "12", "--steps", "3"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert p.returncode == 2 and "CUDA device" in p.stderr
