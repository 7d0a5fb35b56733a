#!/bin/bash
set -u
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_step.py tests/test_gpu_importance.py -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | grep -E "passed|failed|FAILED|outside" | sed "s/^/run $i: /"
done
