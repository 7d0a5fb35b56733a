#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --config c5shard --steps 10 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "rc=$?" >> gpurun_out/c5.err
for i in 1 2; do for v in la0 base la4; do
  if [ $v = base ]; then V=""; else V=$v; fi
  echo "== $v" >> gpurun_out/ab_la.txt
  ASTRA_LIB_VARIANT=$V timeout 200 python scripts/bench_step.py 40 2>&1 | tail -2 >> gpurun_out/ab_la.txt
  ASTRA_LIB_VARIANT=$V timeout 300 python bench.py --emulate 8 --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('emulate8', d['phases_ms_per_step'], d['roofline_step']['launch_ms'])" >> gpurun_out/ab_la.txt
done; done
cat gpurun_out/ab_la.txt; head -c 600 gpurun_out/c5.json; tail -2 gpurun_out/c5.err
