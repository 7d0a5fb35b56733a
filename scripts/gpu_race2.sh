#!/bin/bash
set -u
mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_step.py -m gpu -q -k "adam_matches" -p no:cacheprovider > gpurun_out/san/racecheck2.log 2>&1; echo "rc=$?" >> gpurun_out/san/racecheck2.log
grep -E "Race reported|RACECHECK SUMMARY|passed|failed" gpurun_out/san/racecheck2.log | head
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | grep -E "passed|failed|FAILED|outside" | sed "s/^/full suite $i: /"
done
