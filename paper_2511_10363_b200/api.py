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

    def __init__(self, device: Any = 0, mode: str = "fast", chunk: int = 0,
                 stream: Any = None) -> None:
        """`device`: a CUDA device index, or a sequence of them for a
        multi-device context (psk_create_multi: PKF / PRTS time-sharded over
        the devices, PTFS on their two halves, batches split between them)."""
        L = _lib.lib()
        ctx = C.c_void_p()
        if isinstance(device, (list, tuple)):
            devs = (C.c_int * len(device))(*[int(d) for d in device])
            _check(L.psk_create_multi(C.byref(ctx), devs, len(device)))
            self.devices = [int(d) for d in device]
            device = self.devices[0]
        else:
            _check(L.psk_create(C.byref(ctx), int(device)))
            self.devices = [int(device)]
        self._ctx = ctx
        self.device = int(device)
        self._async = False
        self._pending: list[Any] = []  # marshals alive until sync() (async mode)
        self.set_mode(mode)
        self.set_chunk(chunk)
        if stream is not None:
            self.set_stream(stream)

    def sync(self) -> None:
        """Wait for queued work; raise the first device error since the last
        synchronising call (async mode, option "async")."""
        try:
            _check(_lib.lib().psk_sync(self._ctx))
        finally:
            self._pending.clear()

    def set_option(self, key: str, value: int) -> None:
        _check(_lib.lib().psk_set_option(self._ctx, key.encode(), int(value)))
        if key == "async":
            self._async = bool(value)

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

    def stream_handle(self) -> int:
        """The cudaStream_t the context runs on (psk_get_stream)."""
        h = C.c_void_p()
        _check(_lib.lib().psk_get_stream(self._ctx, C.byref(h)))
        return int(h.value or 0)

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


def _check_out(mk: _Marshal, a: Any, shape: tuple) -> None:
    """A caller-provided output buffer must match the model: shape, dtype,
    C-contiguity and memory kind (CUDA tensors on the inputs' device for a
    device-space model, host memory otherwise) -- the library writes
    shape x dtype bytes of raw row-major data through its pointer."""
    if tuple(a.shape) != shape:
        raise DimensionMismatch(f"output buffer shape {tuple(a.shape)}, expected {shape}")
    if mk.torch:
        import torch
        if not _is_torch(a):
            raise ValueError("outputs must be torch tensors like the inputs")
        if a.dtype != (torch.float64 if mk.f64 else torch.float32):
            raise DimensionMismatch(f"output dtype {a.dtype} differs from the model's")
        if not a.is_contiguous():
            raise ValueError("output buffers must be contiguous")
        if mk.device is not None and a.device != mk.device:
            raise ValueError(f"outputs on {a.device}, inputs on {mk.device}")
        if mk.device is None and a.device.type != "cpu":
            raise ValueError("host-space model: outputs must be host (CPU) tensors")
    else:
        if not isinstance(a, np.ndarray):
            raise ValueError("outputs must be numpy arrays like the inputs")
        if a.dtype != (np.float64 if mk.f64 else np.float32):
            raise DimensionMismatch(f"output dtype {a.dtype} differs from the model's")
        if not a.flags.c_contiguous or not a.flags.writeable:
            raise ValueError("output buffers must be C-contiguous and writeable")


def _outputs(mk: _Marshal, out: GaussianStats | None) -> tuple[Any, Any]:
    if out is None:
        return mk.outputs()
    _check_out(mk, out.mean, (mk.t, mk.nx))
    _check_out(mk, out.cov, (mk.t, mk.nx, mk.nx))
    return out.mean, out.cov


def _ordered_call(bes: list[CudaBackend], mks: list[_Marshal], outs: list[Any], call) -> None:
    """Run `call` (one C-ABI entry) ordered against torch's current stream.

    The contexts run on their own streams.  For device-space (CUDA tensor)
    models their streams first wait for torch's current stream (inputs and the
    contiguous copies _Marshal made are produced there), and torch's stream
    then waits for theirs, so the outputs are ready for torch and memory the
    caching allocator hands out again on torch's stream is not overwritten
    while a queued (async mode) kernel still uses it.  Host marshals of async
    calls are kept alive until sync()."""
    dev = next((mk.device for mk in mks if mk.device is not None), None)
    if dev is None:
        call()
        for be in bes:
            if be._async:
                be._pending.append(mks)
        return
    import torch
    cur = torch.cuda.current_stream(dev)
    if any(len(be.devices) > 1 for be in bes):
        # multi-device calls are synchronous and run on their members' own
        # streams: the inputs must be complete before they start
        cur.synchronize()
        call()
        return
    exts = []
    for be in bes:
        h = be.stream_handle()
        if h not in (cur.cuda_stream, 0):
            ext = torch.cuda.ExternalStream(h, device=torch.device("cuda", be.device))
            ext.wait_stream(cur)
            exts.append(ext)
    call()
    # torch's stream waits for the context's: later torch work on the outputs,
    # and any reuse by the caching allocator of the inputs' / temporaries'
    # memory (allocations on this stream), is ordered after the psk kernels.
    # (No record_stream on the context stream: the allocator would record
    # events on it when the tensors die, possibly after psk_destroy.)
    for ext in exts:
        cur.wait_stream(ext)


def _run(entry: str, m: Lgssm, ys: Any, spec: ScanSpec, be: CudaBackend,
         be_bwd: CudaBackend | None = None, devices: int = 1,
         out: GaussianStats | None = None) -> GaussianStats:
    _validate(m)
    mk = _Marshal(m, ys)
    mean, cov = _outputs(mk, out)
    L = _lib.lib()
    pm = C.c_void_p(mk._ptr(mean))
    pc = C.c_void_p(mk._ptr(cov))
    if entry == "ptfs":
        bes = [be] if be_bwd is None or be_bwd is be else [be, be_bwd]

        def call():
            _check(L.psk_ptfs(be.handle, (be_bwd or be).handle, int(devices),
                              C.byref(mk.model), int(spec.alg), int(spec.sengupta_n), pm, pc))
    else:
        bes = [be]
        fn = L.psk_pkf if entry == "pkf" else L.psk_prts

        def call():
            _check(fn(be.handle, C.byref(mk.model), int(spec.alg), int(spec.sengupta_n),
                      pm, pc))
    _ordered_call(bes, [mk], [mean, cov] if mk.torch else [], call)
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
        mean, cov = _outputs(mk, None if outs is None else outs[i])
        mks.append(mk)
        res.append(GaussianStats(mean, cov))
    devs = {mk.device for mk in mks if mk.device is not None}
    if len(devs) > 1:
        raise ValueError("the device-space series of a batch must share one CUDA device")
    n = len(mks)
    arr = (_lib.psk_model * max(n, 1))(*[mk.model for mk in mks])
    pm = (C.c_void_p * max(n, 1))(*[mks[i]._ptr(res[i].mean) for i in range(n)])
    pc = (C.c_void_p * max(n, 1))(*[mks[i]._ptr(res[i].cov) for i in range(n)])
    fn = _lib.lib().psk_pkf_batch if entry == "pkf" else _lib.lib().psk_prts_batch

    def call():
        _check(fn(be.handle, arr, n, int(spec.alg), int(spec.sengupta_n), pm, pc))
    _ordered_call([be], mks, [], call)
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
