#!/usr/bin/env python
"""Summarise ncu evidence for profiles/: the launch list (per-kernel device
time and share of the step) and the key counters of a `--set full` capture.

usage: python tools/ncu_summary.py <launches.csv> [<prof.ncu-rep>] > profiles/<name>.txt
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_dynamic",
    "sass__inst_executed_register_spilling",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    per: OrderedDict[str, list[float]] = OrderedDict()
    for r in rows[h + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        if d.get("Metric Unit") == "ns":
            v /= 1e3
        elif d.get("Metric Unit") == "ms":
            v *= 1e3
        per.setdefault(name, []).append(v)
    own = {k: v for k, v in per.items() if k.startswith("void psk::") or "psk" in k}
    tot = sum(sum(v) for v in own.values())
    out = ["# launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
           f"{'kernel':70s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}"]
    for k, v in sorted(own.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[:70]:70s} {len(v):8d} {sum(v)/len(v):10.1f} {sum(v)/tot:7.3f}")
    return "\n".join(out)


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = ["# ncu --set full counters"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"## {d.get('Kernel Name', '?')[:110]}")
        out.append(f"grid {d.get('launch__grid_size', '?')} x block {d.get('launch__block_size', '?')}")
        for k in KEYS:
            if k in d:
                out.append(f"{k:80s} {d[k]:>16s} {u.get(k, '')}")
        try:
            rd = float(d["dram__bytes_read.sum"]) * _scale(u["dram__bytes_read.sum"])
            wr = float(d["dram__bytes_write.sum"]) * _scale(u["dram__bytes_write.sum"])
            out.append(f"{'traffic = dram read + write (bytes)':80s} {rd + wr:16.4e}")
        except (KeyError, ValueError):
            pass
    return "\n".join(out)


def _scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
            "GB": 1e9}.get(unit, 1.0)


KNAMES = {"k_filter_reduce": "filter_reduce", "k_filter_finish": "filter_finish_smoother_reduce",
          "k_smoother_finish": "smoother_finish", "k_dlb": "chunk_scan_dlb"}


def traffic_json(path: str, source: str, workload: dict) -> dict:
    """{bench kernel name: {"dram_bytes": read + write per launch}} of a capture"""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "").split("<")[0].split("(")[0].strip().split(" ")[-1]
        key = KNAMES.get(name)
        if key is None:
            continue
        b = float(d["dram__bytes_read.sum"]) * _scale(u["dram__bytes_read.sum"]) + \
            float(d["dram__bytes_write.sum"]) * _scale(u["dram__bytes_write.sum"])
        out[key] = {"dram_bytes": b}
    return {"source": source, "workload": workload, "kernels": out}


if __name__ == "__main__":
    if sys.argv[1] == "--json":  # --json <prof.ncu-rep> <source> <log2t> <dtype> <chunk>
        import json
        print(json.dumps(traffic_json(sys.argv[2], sys.argv[3],
                                      {"log2t": int(sys.argv[4]), "dtype": sys.argv[5],
                                       "chunk": int(sys.argv[6])}), indent=1))
        sys.exit(0)
    if sys.argv[1] == "--full":  # --full <prof.ncu-rep>: the --set full counters only
        print(full(sys.argv[2]))
        sys.exit(0)
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print()
        print(full(sys.argv[2]))
