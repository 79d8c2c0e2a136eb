"""ctypes front-end of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two interchangeable implementations with one Python interface:
  * ``Oracle("port")`` -- oracle/libpsk_oracle.so, our C restatement of the
    reference algorithm (psk_oracle.c; every function cites the reference
    file:line it follows);
  * ``Oracle("ref")``  -- oracle/_ref/libparascan_ref.so, the UNMODIFIED
    reference headers compiled here by oracle/Makefile behind a flat C shim.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "libpsk_oracle.so"
REF_LIB = HERE / "_ref" / "libparascan_ref.so"

ALGS = {"seqscan": 0, "hillis_steele": 1, "blelloch": 2, "inplace_lafi": 3,
        "sengupta_a": 4, "sengupta_b": 5}
# status codes shared with include/psk.h
OK, E_DIM, E_CONTRACT, E_NOT_PD, E_SINGULAR = 0, 1, 2, 3, 4


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


class Flat(C.Structure):
    # `bcast` (port only; the reference shim's struct ends at p0 and never
    # reads it): bit i set = field i of f,u,q,h,d,r,y is one time-invariant block
    _fields_ = [("t", C.c_size_t), ("nx", C.c_int), ("ny", C.c_int)] + [
        (n, C.c_void_p) for n in ("f", "u", "q", "h", "d", "r", "y", "m0", "p0")] + [
        ("bcast", C.c_uint)]

FIELDS = ("f", "u", "q", "h", "d", "r", "y")


def build() -> None:
    """Compile the checkers (the reference shim only when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def dense_fields(m, ys, dtype=np.float64, keep_bcast: bool = False) -> dict:
    """Per-step dense arrays of a model.  Time-invariant fields (no step axis)
    are expanded, or with `keep_bcast` kept as one block and flagged in
    "bcast" (the port reads them with stride 0)."""
    t, nx, ny = int(m.t), int(m.nx), int(m.ny)
    flags = [0]

    def exp(i, a, shp):
        a = np.asarray(a.cpu() if hasattr(a, "cpu") else a, dtype=dtype)
        if a.shape == shp:
            if keep_bcast:
                flags[0] |= 1 << i
                return np.ascontiguousarray(a, dtype=dtype)
            a = np.broadcast_to(a, (t, *shp))
        return np.ascontiguousarray(a, dtype=dtype)

    return dict(
        f=exp(0, m.f, (nx, nx)), u=exp(1, m.u, (nx,)), q=exp(2, m.q, (nx, nx)),
        h=exp(3, m.h, (ny, nx)), d=exp(4, m.d, (ny,)), r=exp(5, m.r, (ny, ny)),
        y=exp(6, ys, (ny,)),
        m0=np.ascontiguousarray(np.asarray(m.prior_mean.cpu() if hasattr(m.prior_mean, "cpu") else m.prior_mean, dtype=dtype)),
        p0=np.ascontiguousarray(np.asarray(m.prior_cov.cpu() if hasattr(m.prior_cov, "cpu") else m.prior_cov, dtype=dtype)),
        t=t, nx=nx, ny=ny, bcast=flags[0])


class Oracle:
    def __init__(self, which: str = "port"):
        self.which = which
        path = PORT_LIB if which == "port" else REF_LIB
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.lib = C.CDLL(str(path))
        self.pre = "pso_" if which == "port" else "psr_"
        if which == "port":
            for n in ("pso_last_scan_work", "pso_last_scan_span", "pso_splitmix64"):
                getattr(self.lib, n).restype = C.c_uint64

    # -- helpers -----------------------------------------------------------
    def _fn(self, name: str, sfx: str | None = None):
        return getattr(self.lib, self.pre + name + (f"_{sfx}" if sfx else ""))

    @staticmethod
    def _flat(fd: dict) -> Flat:
        fl = Flat()
        fl.t, fl.nx, fl.ny = fd["t"], fd["nx"], fd["ny"]
        for n in ("f", "u", "q", "h", "d", "r", "y", "m0", "p0"):
            setattr(fl, n, fd[n].ctypes.data)
        fl.bcast = fd.get("bcast", 0)
        return fl

    @staticmethod
    def _p(a: np.ndarray) -> C.c_void_p:
        return C.c_void_p(a.ctypes.data)

    def _stats(self, fd: dict, dtype):
        return (np.zeros((fd["t"], fd["nx"]), dtype=dtype),
                np.zeros((fd["t"], fd["nx"], fd["nx"]), dtype=dtype))

    def _run(self, what: str, m, ys, dtype, *extra, shim_threads: bool = True):
        dtype = np.dtype(dtype)
        sfx = "d" if dtype == np.float64 else "f"
        fd = dense_fields(m, ys, dtype, keep_bcast=self.which == "port")
        fl = self._flat(fd)
        mean, cov = self._stats(fd, dtype)
        fn = self._fn(what, sfx)
        fn.restype = C.c_int
        args = [C.byref(fl)]
        if what in ("pkf_run", "prts_run", "ptfs_run"):
            alg, sn = extra[0], extra[1]
            args += [C.c_int(alg), C.c_size_t(sn)]
            if self.which == "ref":
                args.append(C.c_uint(extra[2] if len(extra) > 2 else 1))
                if what == "ptfs_run":
                    args.append(C.c_int(extra[3] if len(extra) > 3 else 1))
        args += [self._p(mean), self._p(cov)]
        st = fn(*args)
        if st:
            raise OracleError(st, what)
        return mean, cov

    # -- sequential oracles (kalman_seq.hpp) ----------------------------------
    def kf_run(self, m, ys, dtype=np.float64):
        return self._run("kf_run", m, ys, dtype)

    def rts_run(self, m, ys, dtype=np.float64):
        if self.which == "ref":
            return self._run("rts_run", m, ys, dtype)
        fm, fc = self.kf_run(m, ys, dtype)
        dtype = np.dtype(dtype)
        sfx = "d" if dtype == np.float64 else "f"
        fd = dense_fields(m, ys, dtype, keep_bcast=True)
        fl = self._flat(fd)
        mean, cov = self._stats(fd, dtype)
        st = self._fn("rts_run", sfx)(C.byref(fl), self._p(fm), self._p(fc),
                                      self._p(mean), self._p(cov))
        if st:
            raise OracleError(st, "rts_run")
        return mean, cov

    def tfs_run(self, m, ys, dtype=np.float64):
        return self._run("tfs_run", m, ys, dtype)

    def bif_run(self, m, ys, dtype=np.float64):
        return self._run("bif_run", m, ys, dtype)

    # -- parallel drivers (kalman_par.hpp) -----------------------------------
    def pkf_run(self, m, ys, alg: int, sengupta_n: int = 1, dtype=np.float64, threads=1):
        return self._run("pkf_run", m, ys, dtype, alg, sengupta_n, threads)

    def prts_run(self, m, ys, alg: int, sengupta_n: int = 1, dtype=np.float64, threads=1):
        return self._run("prts_run", m, ys, dtype, alg, sengupta_n, threads)

    def ptfs_run(self, m, ys, alg: int, sengupta_n: int = 1, dtype=np.float64, threads=1,
                 devices=1):
        return self._run("ptfs_run", m, ys, dtype, alg, sengupta_n, threads, devices)

    # -- elements (kalman_elems.hpp) -------------------------------------------
    def make_filter_element(self, m, ys, k: int, dtype=np.float64) -> np.ndarray:
        dtype = np.dtype(dtype)
        sfx = "d" if dtype == np.float64 else "f"
        fd = dense_fields(m, ys, dtype)
        nx = fd["nx"]
        out = np.zeros(3 * nx * nx + 2 * nx, dtype=dtype)
        st = self._fn("make_filter_element", sfx)(C.byref(self._flat(fd)), C.c_size_t(k),
                                                  self._p(out))
        if st:
            raise OracleError(st, "make_filter_element")
        return out

    def filter_combine(self, nx: int, l: np.ndarray, r: np.ndarray) -> np.ndarray:
        sfx = "d" if l.dtype == np.float64 else "f"
        out = np.zeros_like(l)
        st = self._fn("filter_combine", sfx)(C.c_int(nx), self._p(l), self._p(r), self._p(out))
        if st:
            raise OracleError(st, "filter_combine")
        return out

    def make_smoother_element(self, m, ys, fmean_k, fcov_k, k: int, dtype=np.float64):
        dtype = np.dtype(dtype)
        sfx = "d" if dtype == np.float64 else "f"
        fd = dense_fields(m, ys, dtype)
        nx = fd["nx"]
        out = np.zeros(2 * nx * nx + nx, dtype=dtype)
        fm = np.ascontiguousarray(fmean_k, dtype=dtype)
        fc = np.ascontiguousarray(fcov_k, dtype=dtype)
        st = self._fn("make_smoother_element", sfx)(
            C.byref(self._flat(fd)), self._p(fm), self._p(fc), C.c_size_t(k), self._p(out))
        if st:
            raise OracleError(st, "make_smoother_element")
        return out

    def smoother_combine(self, nx: int, l: np.ndarray, r: np.ndarray) -> np.ndarray:
        sfx = "d" if l.dtype == np.float64 else "f"
        out = np.zeros_like(l)
        st = self._fn("smoother_combine", sfx)(C.c_int(nx), self._p(l), self._p(r), self._p(out))
        if st:
            raise OracleError(st, "smoother_combine")
        return out

    def tf_combine(self, x, p, eta, jm):
        sfx = "d" if x.dtype == np.float64 else "f"
        nx = x.shape[0]
        ox = np.zeros_like(x)
        op = np.zeros_like(p)
        st = self._fn("tf_combine", sfx)(C.c_int(nx), self._p(x), self._p(p), self._p(eta),
                                         self._p(jm), self._p(ox), self._p(op))
        if st:
            raise OracleError(st, "tf_combine")
        return ox, op

    # -- generators (model_gen.hpp) ----------------------------------------------
    def gen_model(self, seed: int, nx: int, ny: int, t: int) -> dict:
        a = dict(f=np.zeros((t, nx, nx)), u=np.zeros((t, nx)), q=np.zeros((t, nx, nx)),
                 h=np.zeros((t, ny, nx)), d=np.zeros((t, ny)), r=np.zeros((t, ny, ny)),
                 m0=np.zeros(nx), p0=np.zeros((nx, nx)))
        fn = self.lib[self.pre + "gen_model"]
        st = fn(C.c_uint64(seed), C.c_int(nx), C.c_int(ny), C.c_size_t(t),
                *[self._p(a[k]) for k in ("f", "u", "q", "h", "d", "r", "m0", "p0")])
        if st:
            raise OracleError(st, "gen_model")
        a.update(t=t, nx=nx, ny=ny)
        return a

    def simulate_data(self, g: dict, seed: int) -> np.ndarray:
        fd = dict(g)
        fd["y"] = np.zeros((g["t"], g["ny"]))
        ys = fd["y"]
        fn = self.lib[self.pre + "simulate_data"]
        st = fn(C.byref(self._flat(fd)), C.c_uint64(seed), self._p(ys))
        if st:
            raise OracleError(st, "simulate_data")
        return ys

    # -- scans of the reference's Int64Elems handle ---------------------------
    def int64_scan(self, v: np.ndarray, alg: int, sengupta_n: int = 1, reverse=False):
        v = np.ascontiguousarray(v, dtype=np.int64).copy()
        fn = self.lib[self.pre + "int64_scan"]
        st = fn(C.c_size_t(v.size), self._p(v), C.c_int(alg), C.c_size_t(sengupta_n),
                C.c_int(int(reverse)))
        if st:
            raise OracleError(st, "int64_scan")
        return v

    # -- timing handle (reference only): marshalling excluded ----------------
    def time_handle(self, m, ys, f32: bool = False):
        if self.which != "ref":
            raise RuntimeError("time handles exist for the reference build only")
        fd = dense_fields(m, ys, np.float64)
        fl = self._flat(fd)
        fn = self.lib.psr_handle_create_d
        fn.restype = C.c_void_p
        h = fn(C.byref(fl), C.c_int(int(f32)))
        if not h:
            raise OracleError(-1, "handle_create")
        return _RefHandle(self.lib, h, fd)


class _RefHandle:
    METHODS = {"seq": 0, "pkf": 1, "prts": 2, "ptfs": 3, "kf": 4}

    def __init__(self, lib, h, keep):
        self.lib, self.h, self.keep = lib, h, keep
        lib.psr_handle_time.restype = C.c_double
        lib.psr_handle_time.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_size_t, C.c_uint]

    def time(self, method: str, alg: int = 3, sengupta_n: int = 16, threads: int = 1) -> float:
        s = self.lib.psr_handle_time(self.h, self.METHODS[method], alg, sengupta_n, threads)
        if s < 0:
            raise OracleError(int(s), "handle_time")
        return s

    def __del__(self):
        try:
            self.lib.psr_handle_destroy(C.c_void_p(self.h))
        except Exception:
            pass


class GenModel:
    """Duck-typed Lgssm view over gen_model output (prior under Lgssm names)."""

    def __init__(self, g: dict):
        self.f, self.u, self.q, self.h, self.d, self.r = (g[k] for k in "fuqhdr")
        self.prior_mean, self.prior_cov = g["m0"], g["p0"]
        self.t, self.nx, self.ny = g["t"], g["nx"], g["ny"]
