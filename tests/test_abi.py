"""C-ABI boundary checks that need no GPU: libpsk.so loads, exports every
symbol include/psk.h declares, validates arguments and the reference's scan
contracts before touching a device, and fails loudly (no CPU fallback) when
there is no device.  Also the host-side marshalling of the Python mirror."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import scalar_model

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "psk.h"


def _declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psk_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2511_10363_b200 import _lib
    lib = _lib.lib()
    names = _declared()
    assert len(names) >= 13
    for n in names:
        assert hasattr(lib, n), n
    # the ctypes table covers exactly the header
    assert sorted(_lib.SIGNATURES) == names


def test_version_string():
    from paper_2511_10363_b200 import _lib
    assert b"sm_100a" in _lib.lib().psk_version()


def _model(t=5, nx=1, ny=1, **kw):
    from paper_2511_10363_b200 import api
    m = scalar_model(t) if (nx, ny) == (1, 1) else None
    mk = api._Marshal(m, np.ones((t, 1)))
    for k, v in kw.items():
        setattr(mk.model, k, v)
    return mk


def _call(fn, mk, alg, sn, ctx=None):
    from paper_2511_10363_b200 import _lib
    L = _lib.lib()
    mean, cov = mk.outputs()
    return getattr(L, fn)(ctx, C.byref(mk.model), alg, sn, C.c_void_p(mean.ctypes.data),
                          C.c_void_p(cov.ctypes.data))


def test_validation_without_device():
    from paper_2511_10363_b200 import _lib
    mk = _model(5)
    assert _call("psk_prts", mk, 5, 3) == _lib.PSK_E_CONTRACT      # SenguptaB N=3
    assert b"sengupta_n" in _lib.lib().psk_last_error()
    assert _call("psk_pkf", mk, 9, 1) == _lib.PSK_E_ARG            # unknown alg
    assert _call("psk_pkf", mk, 3, 1) == _lib.PSK_E_ARG            # null context
    bad = _model(5)
    bad.model.nx = 0
    assert _call("psk_pkf", bad, 3, 1) == _lib.PSK_E_DIM           # Mat dims 1..16
    bad.model.nx = 17
    assert _call("psk_pkf", bad, 3, 1) == _lib.PSK_E_DIM
    empty = _model(0)
    assert _call("psk_pkf", empty, 0, 1) == _lib.PSK_E_CONTRACT    # empty Sequential
    assert _call("psk_pkf", empty, 6, 1) == _lib.PSK_E_CONTRACT    # empty DLB
    one = _model(1)
    assert _call("psk_pkf", one, 5, 3) == _lib.PSK_E_ARG           # T=1: no scan check
    assert _lib.lib().psk_ptfs(None, None, 3, C.byref(one.model), 3, 1, None, None) == \
        _lib.PSK_E_ARG                                              # devices in {1,2}


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2511_10363_b200 as psk
    with pytest.raises(psk.CudaError):
        psk.CudaBackend(0)


def test_marshal_strides_and_shapes():
    from paper_2511_10363_b200 import api
    from paper_2511_10363_b200.synthetic import cv_model
    m, ys = cv_model(16, time_varying=True)
    mk = api._Marshal(m, ys)
    assert (mk.model.f_stride, mk.model.y_stride) == (-1, -1)
    assert mk.model.t == 16 and (mk.model.nx, mk.model.ny) == (4, 2)
    mb, _ = cv_model(16, time_varying=False)
    mk = api._Marshal(mb, ys)
    assert mk.model.f_stride == 0 and mk.model.h_stride == 0 and mk.model.y_stride == -1
    mb.f = np.zeros((3, 4, 4))
    with pytest.raises(api.DimensionMismatch):
        api._Marshal(mb, ys)
    m32, ys32 = cv_model(16, dtype=np.float32)
    mk = api._Marshal(m32, ys32)
    assert mk.model.dtype == 0
    with pytest.raises(api.DimensionMismatch):
        api._Marshal(m32, ys)  # mixed dtypes


def test_scan_alg_enum_matches_reference_order():
    """ScanAlg values 0..5 in scan.hpp:32-39 order; DLB appended as 6."""
    from paper_2511_10363_b200 import ScanAlg, to_string
    assert [a.value for a in ScanAlg] == list(range(7))
    assert [to_string(a) for a in list(ScanAlg)[:6]] == [
        "seqscan", "hillis_steele", "blelloch", "inplace_lafi", "sengupta_a", "sengupta_b"]


def test_cpp_shim_header_compiles(tmp_path):
    """include/parascan_b200/cuda_backend.hpp compiles against the reference
    headers (the drop-in overloads of pkf_run / prts_run / ptfs_run)."""
    import shutil
    import subprocess
    ref_inc = Path("/root/reference/proj/core/include")
    if not ref_inc.exists() or not shutil.which("g++"):
        pytest.skip("reference headers not present")
    src = tmp_path / "t.cpp"
    src.write_text('#include "parascan_b200/cuda_backend.hpp"\nint main(){return 0;}\n')
    p = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}",
                        f"-I{ref_inc}", str(src)], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr


def test_batch_validation_without_device():
    """psk_*_batch validate every series (dims, dtype, contracts, outputs)
    before the context is touched, like the single-series entry points."""
    from paper_2511_10363_b200 import _lib
    L = _lib.lib()
    good = _model(5)
    bad = _model(5)
    bad.model.nx = 17
    arr = (_lib.psk_model * 2)(good.model, bad.model)
    outs = [np.empty(5 * 17 * 17) for _ in range(2)]
    pm = (C.c_void_p * 2)(*[C.c_void_p(o.ctypes.data) for o in outs])
    pc = (C.c_void_p * 2)(*[C.c_void_p(o.ctypes.data) for o in outs])
    assert L.psk_prts_batch(None, arr, 2, 6, 1, pm, pc) == _lib.PSK_E_DIM
    arr = (_lib.psk_model * 2)(good.model, good.model)
    assert L.psk_pkf_batch(None, arr, 2, 5, 3, pm, pc) == _lib.PSK_E_CONTRACT  # SenguptaB n=3
    assert L.psk_prts_batch(None, arr, -1, 6, 1, pm, pc) == _lib.PSK_E_ARG
    assert L.psk_prts_batch(None, arr, 2, 6, 1, pm, pc) == _lib.PSK_E_ARG  # null context


def test_out_buffer_validation_without_device():
    """Caller-provided outputs are checked against the model before any
    pointer is taken: dtype, contiguity, kind of memory."""
    import numpy as np

    from paper_2511_10363_b200.api import DimensionMismatch, _check_out, _Marshal
    from paper_2511_10363_b200.synthetic import cv_model

    m, ys = cv_model(8, seed=0)
    mk = _Marshal(m, ys)
    _check_out(mk, np.empty((8, 4)), (8, 4))
    with pytest.raises(DimensionMismatch):
        _check_out(mk, np.empty((8, 4), np.float32), (8, 4))
    with pytest.raises(DimensionMismatch):
        _check_out(mk, np.empty((8, 5)), (8, 4))
    with pytest.raises(ValueError):
        _check_out(mk, np.empty((8, 8))[:, ::2], (8, 4))
    import torch
    with pytest.raises(ValueError):
        _check_out(mk, torch.empty(8, 4, dtype=torch.float64), (8, 4))
