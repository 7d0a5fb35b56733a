#!/bin/bash
# auto sample stride (C5: 64) vs 16, same box; refresh parity at C5
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_refresh_scale.py tests/test_gpu_importance.py -m gpu -q --timeout 500 -p no:cacheprovider -s 2>&1 | grep -E "c5|passed|failed" | head
for i in 1 2; do
for s in auto 16; do
  if [ $s = auto ]; then unset ASTRA_SAMPLE_STRIDE; else export ASTRA_SAMPLE_STRIDE=$s; fi
  timeout 900 python bench.py --config c5shard --no-cpu-baseline --steps 6 > gpurun_out/c5_s$s.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/c5_s$s.json').read().strip().splitlines()[-1])
print('c5 stride=$s', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'gemm', b['roofline']['launch_ms'], 'verify', b['refresh_verify_ms'], b['clocks']['sm_mhz'])"
done
done
unset ASTRA_SAMPLE_STRIDE
