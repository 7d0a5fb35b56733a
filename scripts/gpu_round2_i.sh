#!/bin/bash
set -u
mkdir -p gpurun_out
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "rc=$?" >> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --config dropin --steps 5 > gpurun_out/bench_dropin.json 2> gpurun_out/bench_dropin.err; echo "rc=$?" >> gpurun_out/bench_dropin.err
python - <<'PY'
import json
for c in ("c1", "c2", "c3", "dropin"):
    f = f"gpurun_out/bench_{c}.json"
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
        print(c, b["value"], b["ms_per_step"], b.get("phases_ms_per_step"), b.get("refresh_parity"), (b.get("alt_fp8_refresh") or {}).get("value"), (b.get("e2e") or {}).get("value"), (b.get("cpu_baseline") or {}).get("value"), b.get("refresh_mips_qps"), b["config"].get("l2"))
    except Exception as e:
        print(c, "ERR", e, open(f.replace(".json", ".err")).read()[-1500:])
PY
