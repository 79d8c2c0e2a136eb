#!/usr/bin/env bash
# bench sweep: tools/sweep.sh "<bench args A>" "<bench args B>" ...
mkdir -p gpurun_out
for a in "$@"; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 $a > gpurun_out/sweep.log 2>&1
  python - "$a" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/sweep.log").read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:40s} {d['ms_per_step']:.3f} ms  {d['value']:.3e}  " +
          " ".join(f"{k}={v['avg_ms']:.3f}" for k, v in d["kernels"].items()))
except Exception as e:
    print(sys.argv[1], "FAILED", open("gpurun_out/sweep.log").read()[-500:])
PY
done
