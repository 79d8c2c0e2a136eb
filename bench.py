#!/usr/bin/env python
"""Benchmark: filter + RTS smoother time-steps/s (BASELINE.json metric).

Workload (BASELINE.json configs[3] at N=1): T = 2^24 steps, nx = 4, ny = 2,
FP64, the stationary damped constant-velocity tracking model written per step
(time-varying layout, the reference API is per step), PRTS with the
single-pass decoupled look-back scan.  One "step" of the benchmark is one full
prts_run over the whole series.

  value  -- device-resident throughput: inputs already in HBM, outputs to HBM,
            CUDA events on the library's stream, max over ranks;
  e2e    -- the same PRTS with HOST buffers: at N=1 through the C-ABI with
            pinned host inputs/outputs (H2D of all inputs and D2H of all
            outputs inside the timed region; a stream of series on two async
            contexts so one series' input copy overlaps the previous one's
            result copy); at N>1 every rank copies its shard in from pinned
            host memory, runs the sharded PRTS and copies its shard's result
            out (max over ranks);
  parity -- the output of the last timed step against the CPU oracle's
            sequential kf_run + rts_run (oracle/psk_oracle.c, f64,
            -ffp-contract=off) on the same inputs, over all T steps:
            max |a-b|/(1+|b|) (bench.hpp:216-237), gate 1e-9 FP64 / 1e-4 FP32.

With --gpus N > 1 the time axis is sharded: each rank filters / smooths its
contiguous chunk, the shard aggregates are exchanged with an NCCL all_gather
and folded (paper_2511_10363_b200/distributed.py); scaling is "strong" (T
fixed).  Run without torchrun, `--gpus N` re-launches itself under
torch.distributed.run with N ranks (and fails if fewer GPUs are visible).

--impl reference times the reference's own CPU implementation
(oracle/_ref/libparascan_ref.so: prts_run with PoolBackend on all host
threads) on a bounded sample of the same workload (T = 2^22 by default).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": HBM_FALLBACK, "src": "fallback (B200_PROFILING.md)"}


def _traffic(kernel: str, log2t: int, dtype: str, chunk: int) -> tuple:
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/traffic.json, FP32: traffic_f32.json, written by
    tools/ncu_summary.py --json) when
    it was taken on this workload; (None, None) otherwise."""
    for name in ("traffic.json", "traffic_f32.json"):
        try:
            d = json.loads((ROOT / "profiles" / name).read_text())
            w = d["workload"]
            if w["log2t"] == log2t and w["dtype"] == dtype and w["chunk"] == chunk:
                k = d["kernels"].get(kernel)
                if k is not None:
                    return float(k["dram_bytes"]), d["source"]
        except (OSError, KeyError, ValueError):
            pass
    return None, None


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 5 ms) during the timed
    region; falls back to nvidia-smi polling when NVML is unavailable."""

    REASONS = {  # nvmlClocksEventReason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, index: int):
        self.index = index
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() \
                else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.nv = None
        return self

    def _poll(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            # 5 ms: NVML queries contend with the CUDA driver; polling at 1 kHz
            # stalled the host's kernel launches by milliseconds now and then
            time.sleep(0.005)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


class StreamGate:
    """Holds a stream at a device-memory flag (cuStreamWaitValue32) while the
    host queues the timed steps behind it, then releases it from a second
    stream (cuStreamWriteValue32), so the K steps run back to back on the
    device whatever the host thread does meanwhile.  Host-side stalls during
    the enqueue (NVML clock polling contends with the driver; GIL hand-offs)
    otherwise left the device idle now and then: 5.5 and 15.3 ms/step
    against 4.43 on the same box.  A watchdog releases the gate after 30 s
    in case the enqueue itself ever blocked.  Without cuda-python the timed
    loop runs ungated (gate = False in the JSON line)."""

    def __init__(self, stream, dev):
        import torch
        self.ok = False
        try:
            from cuda.bindings import driver as cu
            self.cu = cu
            self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
            self.rel = torch.cuda.Stream(device=dev)
            self.s = cu.CUstream(stream.cuda_stream)
            self.addr = cu.CUdeviceptr(self.flag.data_ptr())
            self.ok = True
        except Exception:  # noqa: BLE001
            pass
        self._released = threading.Event()

    def close(self) -> None:
        (err,) = self.cu.cuStreamWaitValue32(self.s, self.addr, 1, 0)
        if err != self.cu.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"cuStreamWaitValue32: {err}")
        self._released.clear()
        self._dog = threading.Timer(30.0, self.open)
        self._dog.daemon = True
        self._dog.start()

    def open(self) -> None:
        if self._released.is_set():
            return
        self._released.set()
        self.cu.cuStreamWriteValue32(self.cu.CUstream(self.rel.cuda_stream), self.addr, 1, 0)

    def reset(self) -> None:
        self._dog.cancel()
        self.flag.zero_()


# algorithmic HBM bytes per time step for each fast-path kernel of PRTS
# (DESIGN.md section 4): model inputs 52 scalars (nx=4, ny=2), per-step
# smoothing elements (E, g, upper L) 30 scalars, smoothed stats 20 scalars
def kernel_bytes_per_step(nx: int, ny: int, s: int) -> dict:
    inp = nx * nx * 2 + nx + ny * nx + ny + ny * ny + ny
    st = nx + nx * nx
    egl = nx * nx + nx + nx * (nx + 1) // 2
    return {"filter_reduce": inp * s, "filter_finish_smoother_reduce": (inp + egl) * s,
            "smoother_finish": (egl + st) * s}


def cpu_reference(T_sample: int, threads: int, runs: int, seed: int = 0,
                  per_alg_log2t: int = 20) -> dict:
    """The reference's own CPU path on the same workload (bounded sample):
    prts_run InplaceLaFi on PoolBackend(all host threads), the sequential
    KF + RTS on one core, and every ScanAlg in f64 and f32 (convert_model)
    at a smaller T (bench.hpp:259-323 runs the same matrix)."""
    from oracle.oracle import ALGS, Oracle  # baseline leg only
    from paper_2511_10363_b200.synthetic import cv_model

    m, ys = cv_model(T_sample, seed=seed)
    h = Oracle("ref").time_handle(m, ys)
    h.time("prts", 3, 16, threads)  # warm-up
    ts = [h.time("prts", 3, 16, threads) for _ in range(runs)]
    seq = [h.time("seq", 3, 16, 1) for _ in range(max(1, runs // 3))]
    del h
    tp = 1 << per_alg_log2t
    mp, ysp = cv_model(tp, seed=seed)
    per_alg = {}
    for prec in ("f64", "f32"):
        hp = Oracle("ref").time_handle(mp, ysp, f32=prec == "f32")
        for name, alg in ALGS.items():
            per_alg[f"{name}_{prec}"] = round(tp / hp.time("prts", alg, 16, threads), 1)
        per_alg[f"sequential_kf_rts_1core_{prec}"] = round(tp / hp.time("seq", 3, 16, 1), 1)
        del hp
    return {"value": T_sample * len(ts) / sum(ts), "unit": "time-steps/s",
            "cores": threads, "kind": "reference",
            "sample": f"prts_run InplaceLaFi PoolBackend({threads}) on the first "
                      f"T={T_sample} steps of the same damped-CV f64 workload, "
                      f"median-free mean of {runs} runs after 1 warm-up",
            "sequential_kf_rts_1core": T_sample * len(seq) / sum(seq),
            "per_alg_prts_steps_per_s": per_alg,
            "per_alg_sample": f"T={tp}, one run each, PoolBackend({threads}); "
                              "sequential_* = kf_run + rts_run on 1 core"}


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    T_sample = 1 << args.ref_log2t  # default 2^22: the reference's large-T rate
    from oracle.oracle import Oracle
    from paper_2511_10363_b200.synthetic import cv_model

    m, ys = cv_model(T_sample, seed=0)
    h = Oracle("ref").time_handle(m, ys)
    for _ in range(args.warmup):
        h.time("prts", 3, 16, threads)
    ts = [h.time("prts", 3, 16, threads) for _ in range(args.steps)]
    value = T_sample * len(ts) / sum(ts)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "time-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(ts) / len(ts), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config(args, note=f"reference CPU sample T={T_sample} per step "
                                   f"(the full T=2^{args.log2t} x {args.steps + args.warmup} "
                                   f"runs would take too long on the host)"),
        "cpu_baseline": {"value": value, "unit": "time-steps/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"prts_run InplaceLaFi PoolBackend({threads}), "
                                   f"T={T_sample} per step"},
        "e2e": {"value": value, "unit": "time-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "time-steps/sec filter+smoother (PRTS) vs T, % of HBM roofline"


def config(args, note: str | None = None) -> dict:
    c = {"workload": f"PRTS T=2^{args.log2t} nx=4 ny=2 damped constant-velocity tracking "
                     f"(BASELINE configs[3] at N={args.gpus})",
         "T": 1 << args.log2t, "nx": 4, "ny": 2, "alg": args.alg, "chunk": args.chunk,
         "layout": "per-step (time-varying) model arrays" if not args.broadcast
                   else "time-invariant (broadcast) model, streamed y",
         "l2": "no flush needed: per-step inputs (7.0 GB f64) >> 126 MB L2",
         "parallelism": f"time-sharded x{args.gpus}" if args.gpus > 1 else "single GPU"}
    if note:
        c["note"] = note
    return c


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="psk", choices=["psk", "reference"])
    ap.add_argument("--log2t", type=int, default=24)
    ap.add_argument("--alg", default="DecoupledLookback")
    ap.add_argument("--chunk", type=int, default=0, help="steps per chunk, 0 = auto (one wave)")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--broadcast", action="store_true")
    ap.add_argument("--ref-log2t", type=int, default=22)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-gate", action="store_true",
                    help="enqueue the timed steps while the device runs (no stream gate)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    run_psk(args)


def spawn(args) -> int:
    """`--gpus N` outside torchrun: re-launch this script with N ranks (one
    per GPU, NCCL), as the driver's torchrun launch would."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible",
              file=sys.stderr, flush=True)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


class OracleRun(threading.Thread):
    """The CPU oracle's sequential kf_run + rts_run over the whole series (f64,
    time-invariant blocks read with stride 0), on rank 0 after the timed
    region."""

    def __init__(self, T: int, ys_np: np.ndarray):
        super().__init__(daemon=True)
        self.T, self.ys = T, ys_np
        self.result = None
        self.error = None
        self.seconds = None

    def run(self) -> None:
        try:
            from oracle.oracle import Oracle  # the checker (parity leg only)
            from paper_2511_10363_b200.api import Lgssm
            from paper_2511_10363_b200.synthetic import cv_matrices

            F, Q, H, R, m0, P0 = cv_matrices()
            m = Lgssm(f=F, u=np.zeros(4), q=Q, h=H, d=np.zeros(2), r=R, prior_mean=m0,
                      prior_cov=P0, t=self.T)
            t0 = time.perf_counter()
            self.result = Oracle("port").rts_run(m, self.ys)
            self.seconds = time.perf_counter() - t0
        except Exception as e:  # noqa: BLE001
            self.error = repr(e)


def parity_check(orc, out, lo: int, hi: int, T: int, dev, pg, rank: int, f64: bool) -> dict:
    """max |a-b|/(1+|b|) (bench.hpp:216-237) of the last timed output against
    the oracle over every step; under N ranks rank 0's oracle result is
    broadcast (NCCL) and every rank checks its own shard on its GPU."""
    import torch

    ok = torch.tensor([1.0 if rank != 0 or orc.result is not None else 0.0],
                      device=dev, dtype=torch.float64)
    if pg is not None:
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
    if ok.item() == 0.0:
        return {"error": orc.error if rank == 0 else "oracle failed on rank 0"}
    if rank == 0:
        rm = torch.from_numpy(orc.result[0]).to(dev)
        rc = torch.from_numpy(orc.result[1]).to(dev)
    else:
        rm = torch.empty((T, 4), dtype=torch.float64, device=dev)
        rc = torch.empty((T, 4, 4), dtype=torch.float64, device=dev)
    if pg is not None:
        torch.distributed.broadcast(rm, 0)
        torch.distributed.broadcast(rc, 0)

    def err(got, ref):
        g = got.to(torch.float64)
        return ((g - ref).abs() / (1 + ref.abs())).max()

    e = torch.stack([err(out.mean, rm[lo:hi]), err(out.cov, rc[lo:hi])]).max().reshape(1)
    if pg is not None:
        torch.distributed.all_reduce(e, op=torch.distributed.ReduceOp.MAX)
    tol = 1e-9 if f64 else 1e-4
    res = {"max_rel_err": float(e.item()), "tol": tol, "pass": bool(e.item() <= tol),
           "steps_checked": T, "checked": "smoothed means and covariances of the last "
           "timed step, every time step",
           "oracle": "sequential kf_run + rts_run, oracle/psk_oracle.c (f64, "
                     "-ffp-contract=off; pinned bitwise to the reference), same inputs"}
    if rank == 0 and orc.seconds is not None:
        res["oracle_seconds"] = round(orc.seconds, 1)
    return res


def run_psk(args) -> None:
    import torch

    import paper_2511_10363_b200 as psk
    from paper_2511_10363_b200 import distributed as dist_psk
    from paper_2511_10363_b200.synthetic import cv_matrices, simulate_cv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test rig only (tests/test_gpu_bench_ranks.py): all ranks on one GPU over
    # gloo, to exercise the N > 1 path where NCCL refuses two ranks per GPU
    local = int(os.environ.get("PSK_BENCH_DEVICE", local))
    backend = os.environ.get("PSK_BENCH_DIST_BACKEND", "nccl")
    if world != args.gpus and rank == 0:
        print(f"bench.py: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist.group.WORLD
    T = 1 << args.log2t
    f64 = args.dtype == "f64"
    tdt = torch.float64 if f64 else torch.float32
    S = 8 if f64 else 4
    nx, ny = 4, 2

    # ---- synthetic inputs (same series on every rank; each rank keeps its shard)
    F, Q, H, R, m0, P0 = cv_matrices()
    ys_np = simulate_cv(T, seed=0)
    orc = None
    if not args.no_parity and rank == 0:
        orc = OracleRun(T, ys_np)  # started after the timed region (see below)
    lo, hi = dist_psk.shard_range(T, rank, world)
    hi_in = min(hi + 1, T)  # one extra transition for the smoother boundary

    def field(a, n):
        t = torch.as_tensor(a, dtype=tdt, device=dev)
        if args.broadcast:
            return t
        return t.expand(n, *t.shape).contiguous()

    n_in = hi_in - lo
    model = psk.Lgssm(f=field(F, n_in), u=field(np.zeros(4), n_in), q=field(Q, n_in),
                      h=field(H, n_in), d=field(np.zeros(2), n_in), r=field(R, n_in),
                      prior_mean=torch.as_tensor(m0, dtype=tdt, device=dev),
                      prior_cov=torch.as_tensor(P0, dtype=tdt, device=dev), t=n_in)
    ys = torch.as_tensor(ys_np[lo:hi_in], dtype=tdt, device=dev)
    spec = psk.ScanSpec(psk.ScanAlg[args.alg], 16)
    stream = torch.cuda.Stream(device=dev)
    be = psk.CudaBackend(local, mode="fast", chunk=args.chunk, stream=stream)

    # Device-resident steps are queued back to back ("async": each call returns
    # once its kernels are on the stream; errors and the per-kernel CUDA-event
    # spans are collected by be.sync() after the timed region), so the timed
    # region is GPU time, not host round trips between synchronous calls.
    be.set_option("async", 1)

    def step():
        with torch.cuda.stream(stream):
            out = dist_psk.prts_run_sharded(model, ys, spec, be, rank, world, lo, hi, T, pg)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    be.sync()
    if pg is not None:
        torch.distributed.barrier()
    launches = 0
    prof: dict[str, list[float]] = {}
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    be.set_profile(True)
    out = None
    # (gloo -- the CPU test rig -- blocks the host on CUDA tensors: no gate;
    # under a profiler (ncu serialises every launch: the first gated launch
    # would never return) or with --no-gate the steps run ungated)
    profiled = any(k in os.environ for k in ("CUDA_INJECTION64_PATH", "NV_TPS_LAUNCH_TOKEN",
                                             "NV_NSIGHT_INJECTION_TRANSPORT_TYPE"))
    gate = (StreamGate(stream, dev) if (pg is None or backend == "nccl") and not profiled
            and not args.no_gate else None)
    gated = gate is not None and gate.ok
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if gated:
            gate.close()  # the timed steps queue up behind the gate
        ev0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            out = step()
            launches += be.last_launch_count()
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # enqueue cost per step
        ev1.record(stream)
        if gated:
            gate.open()
        torch.cuda.synchronize()
        if gated:
            gate.reset()
    be.sync()  # raises on any device error of the timed steps
    be.set_profile(False)
    be.set_option("async", 0)
    for name, kms in be.last_profile():
        prof.setdefault(name, []).append(kms)
    ms = ev0.elapsed_time(ev1) / args.steps
    if pg is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = T / (ms * 1e-3)

    # ---- parity of the timed output against the CPU oracle (all T steps)
    parity = None
    if not args.no_parity:
        # The oracle thread is NOT run during the timed region: its Python
        # parts hold the GIL for long stretches, and every ctypes call of the
        # enqueue loop must re-take it -- one run enqueued at 11 ms per step
        # (15.3 ms/step on the device clock instead of 4.43).
        if orc is not None:
            orc.start()
            orc.join()
        with torch.cuda.stream(stream):
            parity = parity_check(orc, out, lo, hi, T, dev, pg, rank, f64)
        torch.cuda.synchronize()
    del out

    # ---- roofline of the dominant kernel (per-launch averages, this run)
    peaks = _peaks()
    bps = kernel_bytes_per_step(nx, ny, S)
    per_kernel = {k: (sum(v) / len(v), len(v)) for k, v in prof.items()}
    totals = {k: sum(v) for k, v in prof.items()}
    dom = max(totals, key=totals.get) if totals else None
    if dom not in bps and totals:  # dominant kernel with an HBM byte model
        dom = max((k for k in totals if k in bps), key=totals.get, default=None)
    steps_local = hi - lo
    roof = None
    if dom in bps:
        avg_ms = per_kernel[dom][0]
        gbs = bps[dom] * steps_local / (avg_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(gbs, 1),
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(gbs / peaks["hbm_gbs"], 4),
                "traffic": _traffic(dom, args.log2t, args.dtype, args.chunk)[0],
                "traffic_source": _traffic(dom, args.log2t, args.dtype, args.chunk)[1],
                "peak_source": peaks["src"],
                "bytes_per_step": bps[dom], "avg_ms": round(avg_ms, 4)}
    kernels = {k: {"avg_ms": round(v[0], 4), "launches_per_step": v[1] // args.steps,
                   "share": round(totals[k] / sum(totals.values()), 4)}
               for k, v in per_kernel.items()}
    for k in kernels:
        if k in bps:
            kernels[k]["GBps"] = round(bps[k] * steps_local / (kernels[k]["avg_ms"] * 1e-3) / 1e9, 1)

    # ---- end to end with host buffers
    e2e = None
    if not args.no_e2e:
        if world == 1:
            e2e = run_e2e(args, psk, T, tdt, F, Q, H, R, m0, P0, ys_np, spec, local)
        else:
            e2e = run_e2e_sharded(args, psk, dist_psk, model, ys, spec, be, stream, rank,
                                  world, lo, hi, T, pg, dev)

    # ---- CPU baseline (reference CPU path, rank 0, N=1 only)
    cpu = None
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        try:
            cpu = cpu_reference(1 << args.ref_log2t, os.cpu_count() or 1, runs=3)
        except Exception as e:  # noqa: BLE001
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic", "config": config(args),
            "roofline": roof, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk.summary(), "kernels": kernels,
            "host_enqueue_ms_per_step": round(host_ms, 3),
            "timing": ("the K steps queued behind a stream gate (cuStreamWaitValue32) and "
                       "released together: CUDA events time device work only" if gated else
                       "steps enqueued while the device runs (no gate)"),
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        torch.distributed.destroy_process_group()


def run_e2e_sharded(args, psk, dist_psk, model, ys, spec, be, stream, rank, world, lo, hi,
                    T, pg, dev) -> dict:
    """N > 1: every rank copies its shard's inputs in from pinned host memory,
    runs the sharded PRTS and copies its shard's smoothed stats out to pinned
    host memory, synchronously, every step; the step time is the max over
    ranks (each rank has its own PCIe link, so the copies scale with N)."""
    import torch

    names = ("f", "u", "q", "h", "d", "r")
    host = {k: torch.empty(getattr(model, k).shape, dtype=getattr(model, k).dtype,
                           pin_memory=True) for k in names}
    for k in names:
        host[k].copy_(getattr(model, k))
    host_y = torch.empty(ys.shape, dtype=ys.dtype, pin_memory=True)
    host_y.copy_(ys)
    n = hi - lo
    hm = torch.empty((n, 4), dtype=ys.dtype, pin_memory=True)
    hc = torch.empty((n, 4, 4), dtype=ys.dtype, pin_memory=True)

    def one():
        with torch.cuda.stream(stream):
            for k in names:
                getattr(model, k).copy_(host[k], non_blocking=True)
            ys.copy_(host_y, non_blocking=True)
            out = dist_psk.prts_run_sharded(model, ys, spec, be, rank, world, lo, hi, T, pg)
            hm.copy_(out.mean, non_blocking=True)
            hc.copy_(out.cov, non_blocking=True)
        stream.synchronize()
        return float(hm[-1, 0])  # the result is on the host

    one()
    steps = max(2, min(args.steps, 8))
    ts = []
    for _ in range(steps):
        torch.distributed.barrier()
        t0 = time.perf_counter()
        one()
        ts.append(time.perf_counter() - t0)
    t = torch.tensor([sum(ts) / len(ts)], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    sec = float(t.item())
    h2d = sum(v.numel() * v.element_size() for v in host.values()) + \
        host_y.numel() * host_y.element_size()
    d2h = hm.numel() * hm.element_size() + hc.numel() * hc.element_size()
    hb = torch.tensor([float(h2d), float(d2h)], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(hb)
    return {"value": T / sec, "unit": "time-steps/s",
            "h2d_bytes_per_step": int(hb[0].item()), "d2h_bytes_per_step": int(hb[1].item()),
            "steps": steps,
            "timer": "wall clock per step (barrier, H2D of the shard, sharded PRTS, D2H of "
                     "the shard's result, host read), max over ranks",
            "pipelining": "none (one synchronous step at a time per rank)"}


def run_e2e(args, psk, T, tdt, F, Q, H, R, m0, P0, ys_np, spec, local) -> dict:
    import torch

    def pinned(a, n=None):
        t = torch.as_tensor(a, dtype=tdt)
        if n is not None and not args.broadcast:
            t = t.expand(n, *t.shape)
        out = torch.empty(t.shape, dtype=tdt, pin_memory=True)
        out.copy_(t)
        return out

    m = psk.Lgssm(f=pinned(F, T), u=pinned(np.zeros(4), T), q=pinned(Q, T),
                  h=pinned(H, T), d=pinned(np.zeros(2), T), r=pinned(R, T),
                  prior_mean=pinned(m0), prior_cov=pinned(P0), t=T)
    ys = pinned(ys_np)
    be = psk.CudaBackend(local, mode="fast", chunk=args.chunk)
    h2d = sum(a.numel() * a.element_size() for a in (m.f, m.u, m.q, m.h, m.d, m.r, ys,
                                                     m.prior_mean, m.prior_cov))
    d2h = T * 20 * (8 if tdt == torch.float64 else 4)
    # pinned outputs, reused across steps (the API call fills them)
    res = psk.GaussianStats(torch.empty((T, 4), dtype=tdt, pin_memory=True),
                            torch.empty((T, 4, 4), dtype=tdt, pin_memory=True))
    psk.prts_run(m, ys, spec, be, out=res)  # warm-up
    ts = []
    steps = max(1, min(args.steps, 5))
    for _ in range(steps):
        t0 = time.perf_counter()
        out = psk.prts_run(m, ys, spec, be, out=res)
        float(out.mean[-1, 0])  # the result is on the host
        ts.append(time.perf_counter() - t0)
    sec_sync = sum(ts) / len(ts)
    # where an end-to-end call goes (CUDA events of one profiled call)
    be.set_profile(True)
    psk.prts_run(m, ys, spec, be, out=res)
    prof = be.last_profile()
    be.set_profile(False)
    br = {"h2d_inputs": sum(ms for n, ms in prof if n == "h2d_inputs"),
          "kernels": sum(ms for n, ms in prof if not n.startswith(("h2d", "d2h"))),
          "d2h_outputs": sum(ms for n, ms in prof if n == "d2h_outputs")}
    # A stream of series through the same API: two contexts in "async" mode
    # take alternate steps, so step i's input copy (H2D) runs while step i-1
    # computes and copies its result back (D2H) -- the two PCIe directions
    # overlap.  Every step still copies its own inputs in and its result out,
    # and the host reads each result after that step's psk_sync.
    bes = [be, psk.CudaBackend(local, mode="fast", chunk=args.chunk)]
    outs = [res, psk.GaussianStats(torch.empty((T, 4), dtype=tdt, pin_memory=True),
                                   torch.empty((T, 4, 4), dtype=tdt, pin_memory=True))]
    for b in bes:
        b.set_option("async", 1)
    for j in range(2):  # warm-up (allocations of the second context)
        psk.prts_run(m, ys, spec, bes[j], out=outs[j])
    for b in bes:
        b.sync()
    psteps = max(4, min(args.steps, 16))  # fill / drain of the 2-deep pipeline amortised
    marks = []
    t0 = time.perf_counter()
    for i in range(psteps):
        j = i % 2
        if i >= 2:
            bes[j].sync()
            float(outs[j].mean[-1, 0])  # step i-2's result, on the host
            marks.append(time.perf_counter() - t0)
        psk.prts_run(m, ys, spec, bes[j], out=outs[j])
    for i in range(psteps - 2, psteps):
        bes[i % 2].sync()
        float(outs[i % 2].mean[-1, 0])
        marks.append(time.perf_counter() - t0)
    sec = (time.perf_counter() - t0) / psteps
    done_ms = [round(1e3 * b, 1) for b in marks]  # when each step's result was on the host
    for b in bes:
        b.set_option("async", 0)
    return {"value": T / sec, "unit": "time-steps/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": psteps,
            "timer": "wall clock over the step loop (host reads every step's result)",
            "pipelining": "2 contexts, async API: step i's H2D overlaps step i-1's "
                          "kernels + D2H",
            "result_on_host_ms": done_ms,
            "sync_value": T / sec_sync,
            "sync_note": "one synchronous call at a time (H2D, kernels, D2H in series)",
            "breakdown_ms": {k: round(v, 2) for k, v in br.items()},
            "pcie_note": "pinned copies: H2D ~55.6 GB/s, D2H ~55.0 GB/s on this box "
                         "(tools/pcie.py); within one PRTS call they cannot overlap (every "
                         "smoothed output depends on every input), across calls they do"}

if __name__ == "__main__":
    main()
