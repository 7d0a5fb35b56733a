#!/bin/bash
# decisive same-box A/B of the refresh layouts (fill=1: 37 parts / 148 SMs; fill=0: 2 parts / 144 SMs, W read once)
set -u
mkdir -p gpurun_out
for i in 1 2 3; do
for f in 1 0; do
  echo "fill=$f $(ASTRA_REFRESH_FILL=$f timeout 300 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep 'bf16 k=96')"
done
done
for i in 1 2 3; do
for f in 1 0; do
  ASTRA_REFRESH_FILL=$f timeout 600 python bench.py --no-cpu-baseline --no-alt-fp8 --steps 10 > gpurun_out/bf$f.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/bf$f.json').read().strip().splitlines()[-1])
print('bench fill=$f', b['value'], b['ms_per_step'], b['phases_ms_per_step']['refresh'], 'gemm', b['roofline']['launch_ms'])"
done
done
for f in 1 0; do
  ASTRA_REFRESH_FILL=$f timeout 900 python bench.py --config c5shard --no-cpu-baseline --steps 6 > gpurun_out/c5f$f.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/c5f$f.json').read().strip().splitlines()[-1])
print('c5 fill=$f', b['value'], b['ms_per_step'], b['phases_ms_per_step']['refresh'], 'gemm', b['roofline']['launch_ms'], b['clocks']['sm_mhz'])"
done
for f in 1 0; do
ASTRA_REFRESH_FILL=$f timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"refresh_tc_kernel" -s 4 -c 1 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep -E "gpu__time|dram__bytes|per_second" | sed "s/^/ncu fill=$f /"
done
