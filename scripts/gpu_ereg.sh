#!/bin/bash
# A/B of the single pass: next-label embedding row in registers (EREG, 4 CTAs/SM: base), without
# (noereg), EREG at 3 CTAs/SM (ereg3); step parity tests on the default; C4 bench for each.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_step.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_step.log
tail -2 gpurun_out/pytest_step.log
for i in 1 2; do
for v in base noereg ereg3; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  echo "== $v"; timeout 300 python scripts/bench_step.py 30 | tail -2
done
done
for v in base noereg ereg3; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1])
print('$v', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'single', b['roofline_step']['kernels']['step_single']['launch_ms'], 'gemm', b['roofline']['launch_ms'], b['clocks']['sm_mhz'])"
done
