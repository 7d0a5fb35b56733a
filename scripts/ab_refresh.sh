#!/bin/bash
# A/B the refresh (k' = 96, 9216 queries, bf16) across library variants: scripts/ab_refresh.sh base v1 ...
for i in 1 2 3; do
for v in "$@"; do
  if [ "$v" = base ]; then echo "== base"; timeout 300 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep "bf16 k";
  else echo "== $v"; ASTRA_LIB_VARIANT=$v timeout 300 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep "bf16 k"; fi
done
done
