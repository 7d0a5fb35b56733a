#!/bin/bash
# Round-2 profiles: launch list of the default bench, ncu --set full of the
# bf16 and e4m3 refresh threshold passes (bench shape), summaries.
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-alt-fp8 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:refresh_tc_kernel -s 4 -c 1 \
  -o gpurun_out/prof_tc_bf16 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-alt-fp8 > gpurun_out/ncu_tc_bf16.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:refresh_tc_kernel -s 4 -c 1 \
  -o gpurun_out/prof_tc_fp8 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --refresh-mode fp8_rerank > gpurun_out/ncu_tc_fp8.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_bench_r02.csv gpurun_out/prof_tc_bf16.ncu-rep gpurun_out/prof_tc_fp8.ncu-rep > gpurun_out/ncu_summary_r02.txt 2>&1
tail -60 gpurun_out/ncu_summary_r02.txt
