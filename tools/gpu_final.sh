#!/usr/bin/env bash
# Round-closing measurement set (run under gpurun; output -> gpurun_out/$1):
# bench lines (FP64 with parity / CPU baseline / e2e, FP32), the ncu launch
# list of the bench command, one ncu --set full capture of the three per-step
# kernels (summary + per-launch DRAM traffic for profiles/traffic.json), and
# BASELINE configs[4] (64 series, nx = 16) in FP64 and FP32.
set -u
O=gpurun_out/${1:-final}
mkdir -p $O
Q="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity --no-gate"
timeout 900 python bench.py > $O/bench_f64.log 2>&1; tail -c 400 $O/bench_f64.log; echo
timeout 900 python bench.py --dtype f32 --no-cpu-baseline > $O/bench_f32.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py $Q > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:k_filter_reduce|k_filter_finish|k_smoother_finish" -s 3 -c 3 -f -o /tmp/prts_prof \
  python bench.py $Q > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/launches.csv /tmp/prts_prof.ncu-rep > $O/ncu_summary.txt 2>&1
python tools/ncu_summary.py --json /tmp/prts_prof.ncu-rep "profiles/$1/ncu_summary.txt" 24 f64 0 \
  > $O/traffic.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:k_filter_reduce|k_filter_finish|k_smoother_finish" -s 3 -c 3 -f -o /tmp/prts_prof32 \
  python bench.py $Q --dtype f32 > $O/ncu_full_f32.log 2>&1
python tools/ncu_summary.py --full /tmp/prts_prof32.ncu-rep > $O/ncu_summary_f32.txt 2>&1
python tools/ncu_summary.py --json /tmp/prts_prof32.ncu-rep "profiles/$1/ncu_summary_f32.txt" 24 f32 0 \
  > $O/traffic_f32.json 2>&1
timeout 900 python tools/config5.py --batch 64 --dtypes f64,f32 --how batch > $O/config5.jsonl 2>&1
ls -la $O
