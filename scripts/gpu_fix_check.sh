#!/bin/bash
# slot-release guard: long GPU suites x3 (the intermittent Adam failure); C2 A/B vs the pre-hot-label library
set -u
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_step.py tests/test_gpu_importance.py tests/test_gpu_encoder_boundary.py tests/test_gpu_full_loss.py -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | grep -E "passed|failed|FAILED|outside" | sed "s/^/suite $i: /"
done
for i in 1 2; do
for v in base prehot; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --config c2 --steps 10 --no-cpu-baseline > gpurun_out/c2_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/c2_$v.json').read().strip().splitlines()[-1])
print('c2 $v', b['value'], b['ms_per_step'], b['phases_ms_per_step'])"
done
done
unset ASTRA_LIB_VARIANT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/launches_c2.csv | head -20
