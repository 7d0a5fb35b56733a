#!/bin/bash
# Full GPU suite repeated until the Adam parity test fails (evidence saved by the test under ASTRA_DIAG_DIR).
mkdir -p gpurun_out/hunt
export ASTRA_DIAG_DIR=gpurun_out/hunt
for i in $(seq 1 12); do
  r=$(timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tee gpurun_out/hunt/run$i.log | grep -E "passed|failed" | tail -1)
  echo "run $i: $r"
  ls gpurun_out/hunt/*.npz >/dev/null 2>&1 && { echo "captured"; break; }
done
