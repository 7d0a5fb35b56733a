#!/bin/bash
# PDL on the sampler too: full GPU suite, smoke, then C4 / C1 / C2 / C3 lines (no CPU baseline).
mkdir -p gpurun_out/pdl2
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pdl2/pytest.log 2>&1; tail -2 gpurun_out/pdl2/pytest.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
for c in c4 c1 c2 c3 c4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/pdl2/$c.json 2>/dev/null
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
b = json.loads(open(f"gpurun_out/pdl2/{c}.json").read().strip().splitlines()[-1])
print(c, b["value"], b["ms_per_step"], b["phases_ms_per_step"], (b.get("e2e") or {}).get("value"), b["clocks"]["sm_mhz"])
PY
done
