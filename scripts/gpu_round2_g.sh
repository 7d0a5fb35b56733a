#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python scripts/fp8_peak.py gpurun_out/fp8_peak.json > gpurun_out/fp8_peak.log 2>&1
timeout 900 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_refresh_scale.py -m gpu -q -s --timeout 600 -p no:cacheprovider -rf > gpurun_out/refresh_tests.log 2>&1; echo "rc=$?" >> gpurun_out/refresh_tests.log
ASTRA_PROFILE_REFRESH=1 timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_fp8_prof.json 2> gpurun_out/bench_fp8_prof.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err
timeout 600 python bench.py --no-cpu-baseline --refresh-mode bf16_rerank > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
cat gpurun_out/fp8_peak.log; grep -E "^\[|passed|failed|rc=|Error" gpurun_out/refresh_tests.log | head -40; grep "refresh stages" gpurun_out/bench_fp8_prof.err | tail -2
python - <<'PY'
import json
for f in ("gpurun_out/bench_fp8.json", "gpurun_out/bench_bf16.json"):
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, b["value"], b["ms_per_step"], b["phases_ms_per_step"], b["refresh_parity"], b["roofline"]["achieved"], b["roofline"]["frac"], b["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-800:])
PY
