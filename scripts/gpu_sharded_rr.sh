#!/bin/bash
# sharded re-rank threshold + Adam single-pass default: tests, emulated N = 2/4/8 (and N = 8 full re-rank), C5
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_step.py tests/test_gpu_importance.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_srr.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_srr.log
tail -3 gpurun_out/pytest_srr.log
for n in 2 4 8; do
  timeout 900 python bench.py --emulate $n --steps 6 > gpurun_out/emulate_${n}gpu.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/emulate_${n}gpu.json').read().strip().splitlines()[-1])
print('N=$n', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline']['launch_ms'])"
done
timeout 900 python bench.py --emulate 8 --emulate-full-rerank --steps 6 > gpurun_out/emulate_8gpu_full.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/emulate_8gpu_full.json').read().strip().splitlines()[-1])
print('N=8 full', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline']['launch_ms'])"
timeout 900 python bench.py --config c5shard --no-cpu-baseline > gpurun_out/bench_c5.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1])
print('c5', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline_step'], b['clocks']['sm_mhz'])"
