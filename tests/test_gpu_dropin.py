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
