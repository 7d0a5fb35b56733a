#!/bin/bash
timeout 150 python -m pytest tests/test_gpu_step.py -q -x -k "schedules_agree" 2>&1 | grep -E "passed|failed|Error|assert|Timeout" | head -8
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,utilization.gpu --format=csv,noheader
for i in 1 2 3; do
echo "== pipe"; ASTRA_STEP_PIPE=1 timeout 60 python scripts/bench_step.py 40 | tail -1
echo "== two-kernel"; timeout 120 python scripts/bench_step.py 40 | tail -1
done
