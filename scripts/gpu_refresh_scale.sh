#!/bin/bash
# Production-size refresh parity (tests/test_gpu_refresh_scale.py) on one B200.
set -u
mkdir -p gpurun_out
(free -g; lscpu | head -20) > gpurun_out/host.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_refresh_scale.py -m gpu -q -s --timeout 1200 -p no:cacheprovider \
  > gpurun_out/refresh_scale.log 2>&1; echo "rc=$?" >> gpurun_out/refresh_scale.log
grep -E "^\[|passed|failed|rc=|Error|assert" gpurun_out/refresh_scale.log | head -40
