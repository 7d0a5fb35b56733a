#!/bin/bash
# launch list (per-launch device time) of the default bench at the current HEAD
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_s3.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-alt-fp8 > gpurun_out/ncu_launch_bench.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_bench_s3.csv > gpurun_out/launches_s3_summary.txt 2>&1
head -40 gpurun_out/launches_s3_summary.txt
