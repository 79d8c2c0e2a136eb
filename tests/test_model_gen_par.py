"""include/parascan_b200/model_gen_par.hpp: the reference's gen_model
(model_gen.hpp:104-158) parallel over steps is BIT-IDENTICAL to the
reference's sequential generator (per-(step, role) streams), for several
seeds and dimensions.  Compiled against the reference headers (present only
in the build container; skipped elsewhere)."""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/core/include")

SRC = r'''
#include <chrono>
#include <cstdio>
#include <cstring>
#include "parascan/model_gen.hpp"
#include "parascan_b200/model_gen_par.hpp"
using namespace parascan;
template <class V> bool same(const V& a, const V& b) {
  if (a.size() != b.size()) return false;
  for (std::size_t k = 0; k < a.size(); ++k) {
    auto x = a[k].view(); auto y = b[k].view();
    if (x.rows != y.rows || x.cols != y.cols ||
        std::memcmp(x.d, y.d, sizeof(double) * x.rows * x.cols)) return false;
  }
  return true;
}
int main() {
  const int cases[][4] = {{0, 4, 2, 5000}, {7, 16, 8, 300}, {123, 1, 1, 1}, {9, 3, 5, 777}};
  for (auto& c : cases) {
    auto a = gen_model(c[0], c[1], c[2], c[3]);
    auto b = gen_model_par(c[0], c[1], c[2], c[3]);
    bool ok = same(a.f, b.f) && same(a.u, b.u) && same(a.q, b.q) && same(a.h, b.h) &&
              same(a.d, b.d) && same(a.r, b.r) &&
              !std::memcmp(a.prior_mean.view().d, b.prior_mean.view().d, 8 * c[1]) &&
              !std::memcmp(a.prior_cov.view().d, b.prior_cov.view().d, 8 * c[1] * c[1]);
    std::printf("seed %d nx %d ny %d T %d: %s\n", c[0], c[1], c[2], c[3], ok ? "identical" : "DIFF");
    if (!ok) return 1;
  }
  const std::size_t T = 1 << 18;
  auto t0 = std::chrono::steady_clock::now();
  auto s = gen_model(1, 4, 2, T);
  auto t1 = std::chrono::steady_clock::now();
  auto p = gen_model_par(1, 4, 2, T);  // first touch of the worker arenas
  t1 = std::chrono::steady_clock::now();
  p = gen_model_par(1, 4, 2, T);
  auto t2 = std::chrono::steady_clock::now();
  std::printf("T=2^18: gen_model %.3f s, gen_model_par %.3f s\n",
              std::chrono::duration<double>(t1 - t0).count(),
              std::chrono::duration<double>(t2 - t1).count());
  return same(s.q, p.q) ? 0 : 1;
}
'''


def test_gen_model_par_bit_identical(tmp_path):
    if not REF_INC.exists() or not shutil.which("g++"):
        pytest.skip("reference headers not present")
    src = tmp_path / "g.cpp"
    src.write_text(SRC)
    exe = tmp_path / "g"
    p = subprocess.run(["g++", "-O2", "-std=c++20", "-pthread", "-ffp-contract=off",
                        f"-I{ROOT / 'include'}", f"-I{REF_INC}", str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
