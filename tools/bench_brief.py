"""One-line summary of a bench.py JSON line on stdin (A/B sweeps):
label, dtype, ms/step, per-kernel average ms."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
ks = sum(v["avg_ms"] * v["launches_per_step"] for v in d["kernels"].values())
print(sys.argv[1] if len(sys.argv) > 1 else "", d["dtype"], round(d["ms_per_step"], 3),
      "kernels", round(ks, 3), "host", d.get("host_enqueue_ms_per_step"),
      {k: v["avg_ms"] for k, v in d["kernels"].items()}, flush=True)
