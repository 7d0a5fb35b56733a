#!/bin/bash
# A/B of the single pass's multi-occurrence scratch: TMEM (default: smem left to the ring, Q=32),
# shared memory with Q=64 (smem: the previous pass), shared memory with Q=32 (smemq32).
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_step.py -m gpu -q -x --timeout 250 -p no:cacheprovider > gpurun_out/pytest_step.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_step.log
tail -2 gpurun_out/pytest_step.log
for i in 1 2; do
for v in base smem smemq32; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  echo "== $v"; timeout 300 python scripts/bench_step.py 30 | tail -1
done
done
for v in base smem; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1])
print('$v', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'single', b['roofline_step']['kernels']['step_single']['launch_ms'], 'gemm', b['roofline']['launch_ms'], b['clocks']['sm_mhz'])"
done
