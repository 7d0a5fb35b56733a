#!/bin/bash
# A/B the bf16 + Adam step microbenchmark across library variants
for i in 1 2; do
for v in "$@"; do
  if [ "$v" = det ]; then echo "== two-kernel"; ASTRA_STEP_SINGLE=0 ASTRA_BENCH_STEP_ADAM=1 timeout 180 python scripts/bench_step.py 30 | tail -2;
  elif [ "$v" = base ]; then echo "== base"; ASTRA_BENCH_STEP_ADAM=1 timeout 180 python scripts/bench_step.py 30 | tail -2;
  else echo "== $v"; ASTRA_LIB_VARIANT=$v ASTRA_BENCH_STEP_ADAM=1 timeout 180 python scripts/bench_step.py 30 | tail -2; fi
done
done
