#!/bin/bash
# same-box A/B: SM-filling refresh layout (37 parts at C4) vs the 93% rule (2 parts, 144 SMs);
# encoder-boundary tests; select launch times under ncu for both
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_encoder_boundary.py tests/test_gpu_refresh.py -m gpu -q --timeout 500 -p no:cacheprovider > gpurun_out/pytest_fill.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_fill.log
tail -3 gpurun_out/pytest_fill.log
for i in 1 2; do
for f in 1 0; do
  ASTRA_REFRESH_FILL=$f timeout 600 python bench.py --no-cpu-baseline --no-alt-fp8 --steps 10 > gpurun_out/bench_fill$f.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/bench_fill$f.json').read().strip().splitlines()[-1])
print('fill=$f', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'gemm', b['roofline']['launch_ms'], b['refresh_parity']['recall_at_k'], b['clocks']['sm_mhz'])"
done
done
for f in 1 0; do
ASTRA_REFRESH_FILL=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select_kernel|refresh_tc|rerank" -c 8 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep -E "^  [a-z].*kernel|gpu__time" | sed 's/(const.*//' | paste - - | awk -v f=$f '{print "fill=" f, $1, $(NF)}'
done
