#!/bin/bash
# A/B the bf16 + Adam single pass (forced) across library variants
for i in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then echo "== base"; ASTRA_STEP_SINGLE_ADAM=1 ASTRA_BENCH_STEP_ADAM=1 timeout 180 python scripts/bench_step.py 30 | tail -1;
  else echo "== $v"; ASTRA_LIB_VARIANT=$v ASTRA_STEP_SINGLE_ADAM=1 ASTRA_BENCH_STEP_ADAM=1 timeout 180 python scripts/bench_step.py 30 | tail -1; fi
done
done
