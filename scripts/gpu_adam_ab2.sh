#!/bin/bash
# single pass: producer back-off 20 ns (base) vs 200 ns (poll200); Adam at 3 CTAs/SM (adam3, +poll200)
set -u
mkdir -p gpurun_out
for i in 1 2; do
for v in base poll200 adam3; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  echo "== $v sgd  $(timeout 300 python scripts/bench_step.py 30 | tail -1)"
  echo "== $v adam $(ASTRA_BENCH_STEP_ADAM=1 timeout 300 python scripts/bench_step.py 30 | tail -1)"
done
done
for v in base poll200 adam3; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  timeout 900 python bench.py --config c5shard --no-cpu-baseline --steps 6 > gpurun_out/c5_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/c5_$v.json').read().strip().splitlines()[-1])
print('c5 $v', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline_step']['kernels'], b['clocks']['sm_mhz'])"
done
