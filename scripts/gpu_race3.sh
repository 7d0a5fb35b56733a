#!/bin/bash
set -u
mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_step.py -m gpu -q -k "adam_matches or bitexact_vs_two" -p no:cacheprovider > gpurun_out/san/racecheck3.log 2>&1; echo "rc=$?" >> gpurun_out/san/racecheck3.log
grep -E "Race reported|Read access|RACECHECK SUMMARY|passed|failed" gpurun_out/san/racecheck3.log | head
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_refresh.py -m gpu -q --timeout 500 -p no:cacheprovider 2>&1 | tail -1
echo "micro sgd  $(timeout 300 python scripts/bench_step.py 30 | tail -1)"
echo "micro adam $(ASTRA_BENCH_STEP_ADAM=1 timeout 300 python scripts/bench_step.py 30 | tail -1)"
timeout 600 python bench.py --no-cpu-baseline --no-alt-fp8 --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('c4', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline_step']['kernels'])"
