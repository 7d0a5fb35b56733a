#!/bin/bash
# test_gpu_step.py repeated with PDL on / off (history-dependent Adam parity failure hunt).
for i in 1 2 3 4 5 6; do
  for pdl in 1 0; do
    r=$(ASTRA_PDL=$pdl timeout 600 python -m pytest tests/test_gpu_step.py -m gpu -q -p no:cacheprovider 2>&1 | grep -E "passed|failed" | tail -1)
    echo "run $i pdl $pdl: $r"
  done
done
