"""Python mirror of the reference's parallel-Kalman API over the CUDA path.

Names, argument meaning and error behaviour follow the reference C++ API:

=====================  =====================================================
this module            reference (/root/reference/proj/core/include/parascan)
=====================  =====================================================
``ScanAlg``            ``enum class ScanAlg`` (scan.hpp:32-39) + the new
                       ``DecoupledLookback`` appended after ``SenguptaB``
``ScanSpec``           ``struct ScanSpec`` (scan.hpp:41-44)
``Lgssm``              ``Lgssm<S>`` (lgssm.hpp:29-42), fields as per-step
                       arrays; a field without the step axis is time-invariant
``GaussianStats``      ``std::vector<GaussianStats<S>>`` (lgssm.hpp:17-21) as
                       two arrays ``mean[T][nx]``, ``cov[T][nx][nx]``
``CudaBackend``        the ``Backend&`` executor slot (backend.hpp:39-44)
``pkf_run``            ``pkf_run`` (kalman_par.hpp:111-119)
``prts_run``           ``prts_run`` (kalman_par.hpp:156-179)
``ptfs_run``           ``ptfs_run`` (kalman_par.hpp:207-238)
exceptions             ``DimensionMismatch``, ``NotPositiveDefinite``,
                       ``SingularMatrix`` (mat.hpp:21-32), ``ContractViolation``
                       (scan.hpp:28-30)
=====================  =====================================================

Inputs may be numpy arrays / CPU tensors (host space: copied in and out by the
library) or CUDA tensors (device space: used in place, outputs returned as
CUDA tensors).  All numerics run in libpsk.so's CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum
from typing import Any

import numpy as np

from . import _lib


class ScanAlg(IntEnum):
    Sequential = 0
    HillisSteele = 1
    Blelloch = 2
    InplaceLaFi = 3
    SenguptaA = 4
    SenguptaB = 5
    DecoupledLookback = 6


_ALG_NAMES = {  # to_string(ScanAlg), scan.hpp:46-56
    ScanAlg.Sequential: "seqscan",
    ScanAlg.HillisSteele: "hillis_steele",
    ScanAlg.Blelloch: "blelloch",
    ScanAlg.InplaceLaFi: "inplace_lafi",
    ScanAlg.SenguptaA: "sengupta_a",
    ScanAlg.SenguptaB: "sengupta_b",
    ScanAlg.DecoupledLookback: "decoupled_lookback",
}


def to_string(a: ScanAlg) -> str:
    return _ALG_NAMES[ScanAlg(a)]


@dataclass(frozen=True)
class ScanSpec:
    alg: ScanAlg = ScanAlg.InplaceLaFi
    sengupta_n: int = 1


class DimensionMismatch(ValueError):
    pass


class ContractViolation(ValueError):
    pass


class NotPositiveDefinite(RuntimeError):
    pass


class SingularMatrix(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERRORS = {
    _lib.PSK_E_DIM: DimensionMismatch,
    _lib.PSK_E_CONTRACT: ContractViolation,
    _lib.PSK_E_NOT_PD: NotPositiveDefinite,
    _lib.PSK_E_SINGULAR: SingularMatrix,
    _lib.PSK_E_CUDA: CudaError,
    _lib.PSK_E_NCCL: CudaError,
    _lib.PSK_E_ARG: ValueError,
    _lib.PSK_E_ALLOC: MemoryError,
}


def _check(status: int) -> None:
    if status != _lib.PSK_OK:
        msg = _lib.lib().psk_last_error().decode()
        raise _ERRORS.get(status, RuntimeError)(msg)


def _is_torch(x: Any) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class Lgssm:
    """Linear-Gaussian state-space model (lgssm.hpp:29-42).

    ``f,u,q`` index k is the transition k -> k+1 (F[0] acts on the prior);
    ``h,d,r`` index k belongs to measurement y[k] (lgssm.hpp:5-8).  Each field
    is either per-step (leading axis T) or time-invariant (no leading axis).
    """

    f: Any
    u: Any
    q: Any
    h: Any
    d: Any
    r: Any
    prior_mean: Any
    prior_cov: Any
    t: int | None = None

    def __post_init__(self) -> None:
        pm = self.prior_mean
        self.nx = int(pm.shape[0])
        h = self.h
        self.ny = int(h.shape[-2])
        if self.t is None:
            ts = [a.shape[0] for a, nd in ((self.f, 3), (self.u, 2), (self.q, 3),
                                          (self.h, 3), (self.d, 2), (self.r, 3))
                  if a.ndim == nd]
            self.t = int(ts[0]) if ts else 0


@dataclass
class GaussianStats:
    mean: Any  # [T][nx]
    cov: Any   # [T][nx][nx]

    def __len__(self) -> int:
        return int(self.mean.shape[0])


class CudaBackend:
    """Executor slot filled by a libpsk context on one CUDA device.

    ``mode`` is ``"fast"`` (chunked kernels, default) or ``"exact"`` (the
    reference's level-by-level kernels in reference operation order).  Like the
    reference's ``PoolBackend`` it must not be driven by two callers at once.
    """

    def __init__(self, device: int = 0, mode: str = "fast", chunk: int = 0,
                 stream: Any = None) -> None:
        L = _lib.lib()
        ctx = C.c_void_p()
        _check(L.psk_create(C.byref(ctx), int(device)))
        self._ctx = ctx
        self.device = int(device)
        self.set_mode(mode)
        self.set_chunk(chunk)
        if stream is not None:
            self.set_stream(stream)

    def sync(self) -> None:
        """Wait for queued work; raise the first device error since the last
        synchronising call (async mode, option "async")."""
        _check(_lib.lib().psk_sync(self._ctx))

    def set_option(self, key: str, value: int) -> None:
        _check(_lib.lib().psk_set_option(self._ctx, key.encode(), int(value)))

    # reference Backend interface: host closures cannot run on the device
    def run(self, launch: Any) -> None:  # backend.hpp:42
        raise ContractViolation("CudaBackend executes only the parallel Kalman "
                                "drivers; host Launch bodies cannot run on it")

    def workers(self) -> int:  # backend.hpp:43
        return 1

    def set_mode(self, mode: str) -> None:
        m = {"fast": _lib.PSK_MODE_FAST, "exact": _lib.PSK_MODE_EXACT}[mode]
        _check(_lib.lib().psk_set_mode(self._ctx, m))
        self.mode = mode

    def set_chunk(self, chunk: int) -> None:
        _check(_lib.lib().psk_set_chunk(self._ctx, int(chunk)))
        self.chunk = int(chunk)

    def set_stream(self, stream: Any) -> None:
        """Run on `stream` (a torch.cuda.Stream or a raw cudaStream_t); None
        restores the context's own stream.  torch's default stream is the
        legacy NULL stream, passed as cudaStreamLegacy (handle 1): a NULL
        handle means "own stream" to the C-ABI."""
        if stream is None:
            handle = 0
        else:
            handle = getattr(stream, "cuda_stream", stream) or 1
        _check(_lib.lib().psk_set_stream(self._ctx, C.c_void_p(handle)))

    def set_profile(self, on: bool) -> None:
        _check(_lib.lib().psk_set_profile(self._ctx, int(bool(on))))

    def last_profile(self) -> list[tuple[str, float]]:
        L = _lib.lib()
        n = L.psk_last_profile(self._ctx, None, None, 0)
        names = (C.c_char_p * max(n, 1))()
        ms = (C.c_float * max(n, 1))()
        L.psk_last_profile(self._ctx, names, ms, n)
        return [(names[i].decode(), float(ms[i])) for i in range(n)]

    def last_launch_count(self) -> int:
        return int(_lib.lib().psk_last_launch_count(self._ctx))

    @property
    def handle(self) -> C.c_void_p:
        return self._ctx

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            _lib.lib().psk_destroy(self._ctx)
            self._ctx = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# marshalling


class _Marshal:
    """Builds a psk_model from an Lgssm + measurements; keeps refs alive."""

    def __init__(self, m: Lgssm, ys: Any) -> None:
        arrays = [m.f, m.u, m.q, m.h, m.d, m.r, ys, m.prior_mean, m.prior_cov]
        torch_in = [_is_torch(a) for a in arrays]
        self.device = None
        if any(torch_in):
            import torch
            devs = {a.device for a, t in zip(arrays, torch_in) if t}
            cuda = [d for d in devs if d.type == "cuda"]
            if cuda and (not all(torch_in) or len(devs) != 1):
                raise ValueError("CUDA inputs must all be CUDA tensors on one device")
            self.device = cuda[0] if cuda else None
            if not all(torch_in):
                arrays = [a if t else torch.as_tensor(np.asarray(a))
                          for a, t in zip(arrays, torch_in)]
            self.torch = True
        else:
            self.torch = False
        dt = arrays[0].dtype
        self.keep = []
        nx, ny, t = m.nx, m.ny, int(m.t)
        self.nx, self.ny, self.t = nx, ny, t
        if self.torch:
            import torch
            if dt not in (torch.float32, torch.float64):
                raise DimensionMismatch(f"unsupported dtype {dt}")
            self.f64 = dt == torch.float64
        else:
            arrays = [np.asarray(a) for a in arrays]
            dt = arrays[0].dtype
            if dt not in (np.float32, np.float64):
                raise DimensionMismatch(f"unsupported dtype {dt}")
            self.f64 = dt == np.float64
        block = [(nx, nx), (nx,), (nx, nx), (ny, nx), (ny,), (ny, ny), (ny,)]
        ptrs, strides = [], []
        for a, shp in zip(arrays[:7], block):
            a = self._prep(a)
            if tuple(a.shape) == shp:
                strides.append(0)
            elif tuple(a.shape) == (t, *shp):
                strides.append(-1)
            else:
                raise DimensionMismatch(f"field shape {tuple(a.shape)} does not match "
                                        f"{shp} or {(t, *shp)}")
            ptrs.append(self._ptr(a))
        pm = self._prep(arrays[7])
        pc = self._prep(arrays[8])
        if tuple(pm.shape) != (nx,) or tuple(pc.shape) != (nx, nx):
            raise DimensionMismatch("prior dims")
        mdl = _lib.psk_model()
        mdl.t = t
        mdl.nx, mdl.ny = nx, ny
        mdl.dtype = _lib.PSK_F64 if self.f64 else _lib.PSK_F32
        mdl.space = _lib.PSK_DEVICE if self.device is not None else _lib.PSK_HOST
        (mdl.f, mdl.u, mdl.q, mdl.h, mdl.d, mdl.r, mdl.y) = ptrs
        (mdl.f_stride, mdl.u_stride, mdl.q_stride, mdl.h_stride, mdl.d_stride,
         mdl.r_stride, mdl.y_stride) = strides
        mdl.prior_mean = self._ptr(pm)
        mdl.prior_cov = self._ptr(pc)
        self.model = mdl

    def _prep(self, a: Any) -> Any:
        if self.torch:
            import torch
            want = torch.float64 if self.f64 else torch.float32
            if a.dtype != want:
                raise DimensionMismatch("all fields must share one dtype")
            a = a.contiguous()
        else:
            want = np.float64 if self.f64 else np.float32
            if a.dtype != want:
                raise DimensionMismatch("all fields must share one dtype")
            a = np.ascontiguousarray(a)
        self.keep.append(a)
        return a

    def _ptr(self, a: Any) -> int:
        return a.data_ptr() if self.torch else a.ctypes.data

    def outputs(self) -> tuple[Any, Any]:
        t, nx = self.t, self.nx
        if self.torch:
            import torch
            dt = torch.float64 if self.f64 else torch.float32
            dev = self.device if self.device is not None else "cpu"
            mean = torch.empty((t, nx), dtype=dt, device=dev)
            cov = torch.empty((t, nx, nx), dtype=dt, device=dev)
        else:
            dt = np.float64 if self.f64 else np.float32
            mean = np.empty((t, nx), dtype=dt)
            cov = np.empty((t, nx, nx), dtype=dt)
        return mean, cov


def _validate(m: Lgssm) -> None:
    if not (1 <= m.nx <= 16 and 1 <= m.ny <= 16):
        raise DimensionMismatch("mat dims")


def _run(entry: str, m: Lgssm, ys: Any, spec: ScanSpec, be: CudaBackend,
         be_bwd: CudaBackend | None = None, devices: int = 1,
         out: GaussianStats | None = None) -> GaussianStats:
    _validate(m)
    mk = _Marshal(m, ys)
    if out is None:
        mean, cov = mk.outputs()
    else:  # caller-provided buffers (e.g. pinned host memory), same kind as inputs
        mean, cov = out.mean, out.cov
        if tuple(mean.shape) != (mk.t, mk.nx) or tuple(cov.shape) != (mk.t, mk.nx, mk.nx):
            raise DimensionMismatch("output buffer shapes")
    L = _lib.lib()
    pm = C.c_void_p(mk._ptr(mean))
    pc = C.c_void_p(mk._ptr(cov))
    if entry == "ptfs":
        st = L.psk_ptfs(be.handle, (be_bwd or be).handle, int(devices),
                        C.byref(mk.model), int(spec.alg), int(spec.sengupta_n), pm, pc)
    else:
        fn = L.psk_pkf if entry == "pkf" else L.psk_prts
        st = fn(be.handle, C.byref(mk.model), int(spec.alg), int(spec.sengupta_n),
                pm, pc)
    _check(st)
    return GaussianStats(mean, cov)


def pkf_run(m: Lgssm, ys: Any, spec: ScanSpec, be: CudaBackend,
            out: GaussianStats | None = None) -> GaussianStats:
    """Parallel Kalman filter, Alg. 5 (kalman_par.hpp:111-119)."""
    return _run("pkf", m, ys, spec, be, out=out)


def prts_run(m: Lgssm, ys: Any, spec: ScanSpec, be: CudaBackend,
             out: GaussianStats | None = None) -> GaussianStats:
    """Parallel RTS smoother, Alg. 6 (kalman_par.hpp:156-179)."""
    return _run("prts", m, ys, spec, be, out=out)


def ptfs_run(m: Lgssm, ys: Any, spec: ScanSpec, be_fwd: CudaBackend,
             be_bwd: CudaBackend | None = None, devices: int = 1,
             out: GaussianStats | None = None) -> GaussianStats:
    """Parallel two-filter smoother, Alg. 7 (kalman_par.hpp:207-238)."""
    return _run("ptfs", m, ys, spec, be_fwd, be_bwd, devices, out=out)


def _run_batch(entry: str, models: list[Lgssm], ys_list: list[Any], spec: ScanSpec,
               be: CudaBackend, outs: list[GaussianStats] | None = None) -> list[GaussianStats]:
    if len(models) != len(ys_list) or (outs is not None and len(outs) != len(models)):
        raise DimensionMismatch("batch lengths differ")
    mks, res = [], []
    for i, (m, ys) in enumerate(zip(models, ys_list)):
        _validate(m)
        mk = _Marshal(m, ys)
        if outs is None:
            mean, cov = mk.outputs()
        else:
            mean, cov = outs[i].mean, outs[i].cov
            if tuple(mean.shape) != (mk.t, mk.nx) or tuple(cov.shape) != (mk.t, mk.nx, mk.nx):
                raise DimensionMismatch("output buffer shapes")
        mks.append(mk)
        res.append(GaussianStats(mean, cov))
    n = len(mks)
    arr = (_lib.psk_model * max(n, 1))(*[mk.model for mk in mks])
    pm = (C.c_void_p * max(n, 1))(*[mks[i]._ptr(res[i].mean) for i in range(n)])
    pc = (C.c_void_p * max(n, 1))(*[mks[i]._ptr(res[i].cov) for i in range(n)])
    fn = _lib.lib().psk_pkf_batch if entry == "pkf" else _lib.lib().psk_prts_batch
    _check(fn(be.handle, arr, n, int(spec.alg), int(spec.sengupta_n), pm, pc))
    return res


def pkf_run_batch(models: list[Lgssm], ys_list: list[Any], spec: ScanSpec, be: CudaBackend,
                  outs: list[GaussianStats] | None = None) -> list[GaussianStats]:
    """A batch of independent series through the PKF (psk_pkf_batch): every
    series validated first, then queued on the context's sub-streams."""
    return _run_batch("pkf", models, ys_list, spec, be, outs)


def prts_run_batch(models: list[Lgssm], ys_list: list[Any], spec: ScanSpec, be: CudaBackend,
                   outs: list[GaussianStats] | None = None) -> list[GaussianStats]:
    """A batch of independent series through the PRTS (psk_prts_batch)."""
    return _run_batch("prts", models, ys_list, spec, be, outs)
