#!/usr/bin/env bash
# One GPU session (run under gpurun): parity tests, smoke, bench, launch list,
# one ncu --set full capture of the dominant kernel.  Output -> gpurun_out/.
# Usage: tools/gpu_check.sh [tests|smoke|bench|ncu|all]...
set -u
O=gpurun_out
mkdir -p $O
what="${*:-all}"
has() { [[ " $what " == *" $1 "* || " $what " == *" all "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active \
  --format=csv > $O/smi_start.csv 2>&1
if has tests; then
  timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 > $O/pytest_gpu.log 2>&1
  echo "rc=$?" >> $O/pytest_gpu.log
  tail -5 $O/pytest_gpu.log
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
  echo "rc=$?" >> $O/smoke.log
  tail -3 $O/smoke.log
fi
if has bench; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $O/bench.log 2>&1
  echo "rc=$?" >> $O/bench.log
  tail -3 $O/bench.log
fi
if has ncu; then
  NCU_ARGS="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-}"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py $NCU_ARGS > $O/ncu_launches.log 2>&1
  echo "rc=$?" >> $O/ncu_launches.log
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:${NCU_KERNEL:-k_filter_reduce|k_filter_finish|k_smoother_finish}" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-3} -f -o $O/prof \
    python bench.py $NCU_ARGS > $O/ncu_full.log 2>&1
  echo "rc=$?" >> $O/ncu_full.log
  tail -3 $O/ncu_full.log
fi
