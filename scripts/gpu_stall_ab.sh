#!/bin/bash
# Host-stall diagnosis of the short-step lines (C2/C3): per-step sampler intervals with the
# nvidia-smi clock poll at 20 ms (default), 100 ms and 500 ms; plus the new engine snapshot GPU test.
mkdir -p gpurun_out/stall
timeout 300 python -m pytest tests/test_engine_snapshot.py -q -m gpu -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
for ms in 20 100 500; do
  for c in c3 c2; do
    ASTRA_BENCH_PHASE_DUMP=1 ASTRA_BENCH_SMI_MS=$ms timeout 300 python bench.py --config $c --no-cpu-baseline \
      > gpurun_out/stall/${c}_smi${ms}_r$rep.json 2> gpurun_out/stall/${c}_smi${ms}_r$rep.err
    python - "$c" "$ms" "$rep" <<'PY'
import json, sys
c, ms, rep = sys.argv[1:]
b = json.loads(open(f"gpurun_out/stall/{c}_smi{ms}_r{rep}.json").read().strip().splitlines()[-1])
big = [l.strip() for l in open(f"gpurun_out/stall/{c}_smi{ms}_r{rep}.err") if l.startswith("step") and any(float(x) > 0.3 for x in l.split("[")[1].rstrip("]\n").split(","))]
print(c, "smi", ms, "rep", rep, b["value"], b["ms_per_step"], b["phases_ms_per_step"], "stalled steps:", len(big), big[:3])
PY
  done
done
done
