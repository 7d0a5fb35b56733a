#!/bin/bash
set -u
mkdir -p gpurun_out
cp gpurun_out/fp8_peak.json profiles/fp8_peak.json 2>/dev/null
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest "tests/test_gpu_refresh.py::test_quantize_e4m3_matches_torch" "tests/test_gpu_refresh.py::test_fp8_rerank_equals_fp32" -m gpu -q -x --timeout 200 -p no:cacheprovider -rf > gpurun_out/fp8_small.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/fp8_small.log
tail -30 gpurun_out/fp8_small.log
if [ $rc -ne 0 ]; then exit 0; fi
timeout 900 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_refresh_scale.py -m gpu -q -s --timeout 600 -p no:cacheprovider -rf > gpurun_out/refresh_tests.log 2>&1; echo "rc=$?" >> gpurun_out/refresh_tests.log
ASTRA_PROFILE_REFRESH=1 timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_fp8_prof.json 2> gpurun_out/bench_fp8_prof.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err
grep -E "^\[|passed|failed|rc=" gpurun_out/refresh_tests.log | head -40; grep "refresh stages" gpurun_out/bench_fp8_prof.err | tail -2
python - <<'PY'
import json
for f in ("gpurun_out/bench_fp8.json",):
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, b["value"], b["ms_per_step"], b["phases_ms_per_step"], b["refresh_parity"], b["roofline"], b["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-800:])
PY
