#!/bin/bash
# A/B of the refresh sample-pass tile stride (ASTRA_SAMPLE_STRIDE) inside the C4 bench.
mkdir -p gpurun_out
for s in ${STRIDES:-16 32 24 16 32}; do
  echo "== stride $s"
  ASTRA_SAMPLE_STRIDE=$s timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print(r['value'], r['e2e']['value'], r['phases_ms_per_step'], 'verify', r['refresh_verify_ms'])"
done
