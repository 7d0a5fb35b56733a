#!/bin/bash
# hot labels out of the single pass: step parity, the C4 uniform and clustered lines, C5
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_encoder_boundary.py tests/test_gpu_importance.py -m gpu -q -x --timeout 500 -p no:cacheprovider > gpurun_out/pytest_hot.log 2>&1; rc=$?
tail -2 gpurun_out/pytest_hot.log
if [ $rc -ne 0 ]; then grep -E "Error|assert|FAILED" gpurun_out/pytest_hot.log | head -20; exit 0; fi
echo "micro $(timeout 300 python scripts/bench_step.py 30 | tail -1)"
for w in clustered uniform; do
  timeout 600 python bench.py --w-init $w --no-cpu-baseline --no-alt-fp8 --steps 10 > gpurun_out/bench_$w.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1])
print('$w', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'verify_ms', b['refresh_verify_ms'], 'single', b['roofline_step']['kernels'].get('step_single'), b['refresh_parity']['recall_at_k'])"
done
timeout 900 python bench.py --config c5shard --no-cpu-baseline --steps 6 > gpurun_out/bench_c5.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1])
print('c5', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline_step']['kernels'], b['clocks']['sm_mhz'])"
