#!/bin/bash
set -u
mkdir -p gpurun_out
for s in 1 0; do
  ASTRA_STEP_SINGLE_ADAM=$s timeout 300 python -m pytest tests/test_gpu_step.py -m gpu -q --timeout 250 -p no:cacheprovider -k "adam" 2>&1 | tail -3 | sed "s/^/single_adam=$s alone: /"
done
timeout 600 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_step.py -m gpu -q --timeout 500 -p no:cacheprovider -k "rerank_candidates or adam_matches" 2>&1 | tail -3 | sed "s/^/after rerank test: /"
timeout 600 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_step.py -m gpu -q --timeout 500 -p no:cacheprovider -k "not rerank_candidates" 2>&1 | tail -3 | sed "s/^/without rerank test: /"
