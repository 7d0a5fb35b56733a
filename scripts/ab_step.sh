#!/bin/bash
# A/B the step microbenchmark across library variants: scripts/ab_step.sh base v1 v2 ...
for i in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then echo "== base"; timeout 120 python scripts/bench_step.py 40 | tail -2;
  else echo "== $v"; ASTRA_LIB_VARIANT=$v timeout 120 python scripts/bench_step.py 40 | tail -2; fi
done
done
