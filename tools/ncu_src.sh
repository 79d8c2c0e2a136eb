#!/usr/bin/env bash
# Source-level (SASS) stall attribution of the per-step kernels of one
# bench.py configuration (run under gpurun; output -> gpurun_out/$1):
# ncu --set full with source counters, one capture per kernel, exported on
# the box as the raw page and the SASS source page (CSV; the .ncu-rep files
# are too large to bring back).  $2 = dtype, $3 = kernel regex.
set -u
O=gpurun_out/${1:-src}
D=${2:-f64}
K=${3:-k_filter_reduce|k_filter_finish|k_smoother_finish}
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s ${4:-3} -c ${5:-3} -f \
  -o /tmp/src_prof python bench.py --dtype $D --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  --no-parity --no-gate > $O/ncu_$D.log 2>&1
ncu -i /tmp/src_prof.ncu-rep --page raw --csv > $O/${D}_raw.csv 2>&1
for k in $(echo $K | tr '|' ' '); do
  ncu -i /tmp/src_prof.ncu-rep -k "regex:$k" --page source --csv --print-source sass \
    > $O/${D}_src_$k.csv 2>&1
done
ls -la $O
