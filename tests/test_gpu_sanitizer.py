"""compute-sanitizer over the fast path (every ScanAlg incl. the decoupled
look-back's flag protocol, the tile sweeps, the TMA-staged passes and the
wide path): the GPU analogue of the reference's WriteSetRecorderBackend race
detector (backend.hpp:134-151).  memcheck (out-of-bounds /
misaligned accesses), racecheck (shared-memory hazards) and synccheck
(barrier misuse) must report 0 errors."""
from __future__ import annotations

import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(gpu, tool):
    if not Path(SAN).exists():
        pytest.skip("compute-sanitizer not found")
    p = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        str(ROOT / "tools" / "sanitize_case.py")],
                       capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "sanitize case done" in out
