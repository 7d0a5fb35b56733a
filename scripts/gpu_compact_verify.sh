#!/bin/bash
# compact verify: refresh parity (incl. forced verify, clustered, C5), the C4 line and the clustered C4 line
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_refresh.py -m gpu -q -x --timeout 250 -p no:cacheprovider > gpurun_out/pytest_cv1.log 2>&1; rc=$?
tail -2 gpurun_out/pytest_cv1.log
if [ $rc -ne 0 ]; then grep -E "Error|assert" gpurun_out/pytest_cv1.log | head -20; exit 0; fi
timeout 900 python -m pytest tests/test_gpu_refresh_scale.py tests/test_gpu_importance.py tests/test_dropin_train_golden.py -m gpu -q --timeout 800 -p no:cacheprovider -s 2>&1 | grep -E "flagged|recall|passed|failed|Error" | head -30
for w in clustered uniform; do
  timeout 600 python bench.py --w-init $w --no-cpu-baseline --steps 10 > gpurun_out/bench_$w.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1])
print('$w', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'verify_ms', b['refresh_verify_ms'], b['refresh_parity'], 'gemm', b['roofline']['launch_ms'])"
done
