#!/bin/bash
# step changes: step parity tests, the step microbenchmarks (SGD, bf16+Adam), C4 + C5 bench lines
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_sampler.py tests/test_gpu_importance.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_step.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_step.log
timeout 300 python scripts/bench_step.py 30 > gpurun_out/micro_sgd.txt 2>&1
ASTRA_BENCH_STEP_ADAM=1 timeout 300 python scripts/bench_step.py 30 > gpurun_out/micro_adam.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --config c5shard --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
tail -3 gpurun_out/pytest_step.log; tail -2 gpurun_out/micro_sgd.txt gpurun_out/micro_adam.txt
python - <<'PY'
import json
for f in ("gpurun_out/bench.json", "gpurun_out/bench_c5.json"):
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, b["value"], b["ms_per_step"], b.get("phases_ms_per_step"), b["roofline"]["launch_ms"], b["roofline"]["frac"], b.get("roofline_step"), b.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
