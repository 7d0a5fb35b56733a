#!/bin/bash
# One ncu --set full capture of the refresh_tc kernel (bf16 top-k, k'=96, 9216 queries x 1.3M labels).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:refresh_tc_kernel -s ${SKIP:-4} -c 1 \
  -o gpurun_out/prof_tc_${TAG:-x} python scripts/bench_refresh_k.py 9216 96 > gpurun_out/ncu_tc_${TAG:-x}.log 2>&1
tail -3 gpurun_out/ncu_tc_${TAG:-x}.log
