#!/usr/bin/env bash
# Reference-schema CSV rows from the GPU (run under gpurun; output -> gpurun_out/):
# BASELINE configs[0] (CPU oracle run: the reference's own rows at T = 2^12),
# configs[1] (T sweep, every ScanAlg, f64 and f32, max_rel_err vs the f64
# sequential oracle, device steps/s and roofline fractions) and the drop-in's
# host marshalling cost (wall vs device time, 1 vs all host threads).
set -u
O=gpurun_out
mkdir -p $O
B=tools/_bin/psk_bench
timeout 600 $B run --backend pool --model cv --T 4096 --methods prts pkf ptfs seq_kf seq_rts \
  --algs all --precision f64 --runs 5 --warmup 1 --threads $(nproc) --out $O/csv_config1_reference.csv \
  > /dev/null 2> $O/csv_config1.err
for p in f64 f32; do
  timeout 1500 $B run --model cv --T 1024 16384 262144 1048576 4194304 --methods pkf prts ptfs \
    --algs all --precision $p --runs 5 --warmup 1 --out $O/csv_config2_$p.csv > /dev/null 2> $O/csv_config2_$p.err
done
for th in 1 $(nproc); do
  timeout 900 $B run --model cv --T 4194304 --methods prts --precision f64 --runs 4 --warmup 1 \
    --threads $th --out $O/csv_marshal_t$th.csv > /dev/null 2> $O/csv_marshal_t$th.err
done
timeout 900 $B run --backend pool --model cv --T 4194304 --methods prts --precision f64 --runs 2 \
  --warmup 1 --threads $(nproc) --out $O/csv_marshal_reference.csv > /dev/null 2> $O/csv_marshal_ref.err
ls -la $O/*.csv
