#!/bin/bash
# refresh layout check: refresh parity tests + the C4 bench line (+ C5 shard)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_refresh.py tests/test_gpu_refresh_scale.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_refresh.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_refresh.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --config c5shard --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
tail -3 gpurun_out/pytest_refresh.log
python - <<'PY'
import json
for f in ("gpurun_out/bench.json", "gpurun_out/bench_c5.json"):
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, b["value"], b["ms_per_step"], b.get("phases_ms_per_step"), b.get("refresh_parity"), b["roofline"]["launch_ms"], b["roofline"]["frac"], (b.get("alt_fp8_refresh") or {}).get("value"), b.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
