#!/bin/bash
# Refresh kernel sweep: cluster size x (top-k on/off); one process per setting.
mkdir -p gpurun_out
for cl in 1 2 4; do
  for nt in 0 1; do
    if [ "$nt" = 1 ]; then export ASTRA_TC_DEBUG_NO_TOPK=1; else unset ASTRA_TC_DEBUG_NO_TOPK; fi
    echo "== CL=$cl NO_TOPK=$nt"
    ASTRA_TC_CLUSTER=$cl timeout 300 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep -v cuBLAS
  done
done
unset ASTRA_TC_DEBUG_NO_TOPK
timeout 300 python scripts/bench_refresh_k.py 9216 96 2>&1 | grep cuBLAS
