"""ChunkOrder (psk_common.cuh): the slot map of chunk-element buffers scanned
by the decoupled look-back.  For every n, per and direction it must send the
n chunks to distinct slots below cap(), follow the scan order tile by tile,
and place look-back thread t's per consecutive elements at j * 128 + t.
Host-compiled with g++ against the CUDA headers (no device needed)."""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA_INC = Path("/usr/local/cuda/include")

SRC = r'''
#include <cstdio>
#include <vector>
#include "psk_common.cuh"
using psk::ChunkOrder;
int main() {
  const long long ns[] = {1, 2, 127, 128, 129, 511, 512, 513, 1000, 4096, 151147};
  for (long long n : ns)
    for (int per = 0; per <= 5; ++per)
      for (int rev = 0; rev < 2; ++rev) {
        const ChunkOrder o{n, per, rev};
        const long long cap = o.cap();
        if (cap < n) { std::printf("cap < n\n"); return 1; }
        std::vector<char> seen((size_t)cap, 0);
        for (long long c = 0; c < n; ++c) {
          const long long q = o.at(c);
          if (q < 0 || q >= cap || seen[(size_t)q]) {
            std::printf("n=%lld per=%d rev=%d c=%lld -> %lld\n", n, per, rev, c, q);
            return 1;
          }
          seen[(size_t)q] = 1;
          if (per > 0) {  // scan element g = t per + j of its tile -> j 128 + t
            const long long g = rev ? n - 1 - c : c;
            const long long tile = 128LL * per, r = g % tile;
            if (q != g / tile * tile + (r % per) * 128 + r / per) return 2;
          } else if (q != c) {
            return 3;
          }
        }
      }
  std::printf("ok\n");
  return 0;
}
'''


def test_chunk_order_is_injective_and_tile_transposed(tmp_path):
    if not shutil.which("g++") or not CUDA_INC.exists():
        pytest.skip("g++ or CUDA headers absent")
    src = tmp_path / "co.cpp"
    src.write_text(SRC)
    exe = tmp_path / "co"
    p = subprocess.run(["g++", "-std=c++17", "-O1", "-x", "c++", f"-I{CUDA_INC}",
                        f"-I{ROOT / 'paper_2511_10363_b200' / 'csrc'}", str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr[-3000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
