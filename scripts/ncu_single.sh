#!/bin/bash
# Parity of the step tests + one ncu --set full capture of step_single_tma at the bench shape.
mkdir -p gpurun_out
#timeout 600 python -m pytest tests/test_gpu_step.py -q 2>&1 | grep -E "^E  .*Error|passed|failed|^FAILED" | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_single" -s 3 -c 1 \
  -o gpurun_out/prof_single_${TAG:-x} python scripts/bench_step.py 3 > gpurun_out/ncu_single.log 2>&1
tail -2 gpurun_out/ncu_single.log
