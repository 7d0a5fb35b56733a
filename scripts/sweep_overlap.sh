#!/bin/bash
# bench.py value vs the refresh SM budget (0 = serial refresh then training)
for n in 0 72 88 104 120 136 148; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --refresh-sms $n 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('sms=$n value=%.0f ms=%.2f phases=%s e2e=%.0f gemm_ms=%.2f' % (d['value'], d['ms_per_step'], d['phases_ms_per_step'], d['e2e']['value'], d['roofline']['launch_ms']))"
done
