"""Build libpsk.so (the CUDA kernels + C-ABI) in-tree for sm_100a.

Four translation units are compiled in parallel:
  psk_capi.cu   C-ABI, validation, marshalling (host side)
  psk_fast_f32.cu / psk_fast_f64.cu  fast chunked kernels (FMA on)
  psk_exact.cu  exact reference-order kernels (--fmad=false)
The result lands in paper_2511_10363_b200/lib/libpsk.so (git-ignored, shipped
to the GPU box with the tree).
"""
from __future__ import annotations

import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
OBJ = PKG / "lib" / "obj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
                 "-I", str(PKG.parent / "include"), "--expt-relaxed-constexpr"]
UNITS = {
    "psk_capi.cu": [],
    "psk_fast_f32.cu": [],
    "psk_fast_f64.cu": [],
    "psk_exact.cu": ["--fmad=false"],
    "psk_tile_f32.cu": [],
    "psk_tile_f64.cu": [],
}


_INC = re.compile(r'^\s*#\s*include\s+"([^"]+)"', re.M)


def _deps(src: Path, seen: set | None = None) -> set:
    """The quoted includes of src, transitively (local headers only)."""
    seen = set() if seen is None else seen
    if src in seen or not src.exists():
        return seen
    seen.add(src)
    for name in _INC.findall(src.read_text(errors="replace")):
        _deps((src.parent / name).resolve(), seen)
    return seen


def _needs(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in _deps(src.resolve()))


def _compile(unit: str, extra: list[str], verbose: bool) -> tuple[str, int, str]:
    src = CSRC / unit
    obj = OBJ / (unit + ".o")
    if not _needs(obj, src):
        return unit, 0, "up to date"
    cmd = [NVCC, *COMMON, *extra, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    return unit, p.returncode, p.stdout + p.stderr


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    units = {u: e for u, e in UNITS.items() if (CSRC / u).exists()}
    with ThreadPoolExecutor(max_workers=len(units)) as ex:
        results = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose), units.items()))
    for unit, rc, log in results:
        if rc != 0:
            raise RuntimeError(f"nvcc failed for {unit}:\n{log}")
        if verbose and log.strip():
            print(f"== {unit}\n{log}")
    out = LIB / "libpsk.so"
    objs = [str(OBJ / (u + ".o")) for u in units]
    if not out.exists() or any(Path(o).stat().st_mtime > out.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(out), *objs, "-lcudart_static",
               "-lrt", "-ldl", "-lpthread"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stdout}{p.stderr}")
    # measurement tools (FMA peak, chunk-walk memory patterns): not the product
    tools = LIB / "libpsk_tools.so"
    srcs = [CSRC / "psk_peak.cu", CSRC / "psk_membench.cu"]
    deps = srcs + [CSRC / "psk_stage.cuh", CSRC / "psk_mat.cuh"]
    if not tools.exists() or any(d.stat().st_mtime > tools.stat().st_mtime for d in deps):
        cmd = [NVCC, *COMMON, "-shared", "-o", str(tools), *map(str, srcs)]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"tools build failed:\n{p.stdout}{p.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
