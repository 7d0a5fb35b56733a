#!/bin/bash
# select cursor + device-resident drop-in slates: refresh + drop-in tests, C4 and drop-in bench lines
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_refresh_scale.py tests/test_dropin_cuda.py tests/test_dropin_train_golden.py -m gpu -q --timeout 800 -p no:cacheprovider > gpurun_out/pytest_sd.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_sd.log
tail -3 gpurun_out/pytest_sd.log
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('c4', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'gemm', b['roofline']['launch_ms'], b['refresh_parity'], b['clocks']['sm_mhz'])"
timeout 900 python bench.py --config dropin --steps 5 > gpurun_out/bench_dropin.json 2> gpurun_out/bench_dropin.err
tail -1 gpurun_out/bench_dropin.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_kernel -c 3 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep -E "select_kernel|gpu__time" | head -8
