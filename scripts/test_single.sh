#!/bin/bash
# single label-major pass: parity + A/B timing against the two-kernel schedule
timeout 600 python -m pytest tests/test_gpu_step.py -q 2>&1 | grep -E "^E  .*Error|passed|failed|^FAILED" | head -30
for i in 1 2; do
echo "== single"; timeout 120 python scripts/bench_step.py 40 | tail -2
echo "== two-kernel"; ASTRA_STEP_SINGLE=0 timeout 120 python scripts/bench_step.py 40 | tail -2
done
