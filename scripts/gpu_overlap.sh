#!/bin/bash
# refresh on a side stream under an SM budget, concurrently with the training minibatches (the
# reference's background _RefreshJob), vs serial; same box
set -u
mkdir -p gpurun_out
for n in 0 148 132 120 104 0; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-alt-fp8 --refresh-sms $n > gpurun_out/ov_$n.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ov_$n.json').read().strip().splitlines()[-1])
print('sms=$n value=%.0f ms=%.2f phases=%s gemm_ms=%.2f e2e=%.0f clk=%s' % (d['value'], d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['launch_ms'], d['e2e']['value'], d['clocks']['sm_mhz']))"
done
