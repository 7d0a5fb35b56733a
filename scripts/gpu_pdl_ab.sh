#!/bin/bash
# PDL on the step's kernel chain: full GPU suite, then A/B (ASTRA_PDL=1 vs 0) of C4 / C1 / C2,
# then the C3 line with its CPU baseline and the per-step phase dump (stall diagnosis).
mkdir -p gpurun_out/pdl
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pdl/pytest.log 2>&1; tail -2 gpurun_out/pdl/pytest.log
for rep in 1 2; do
  for pdl in 1 0; do
    for c in c4 c1 c2; do
      ASTRA_PDL=$pdl timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/pdl/${c}_pdl${pdl}_r$rep.json 2>/dev/null
      python - $c $pdl $rep <<'PY'
import json, sys
c, p, r = sys.argv[1:]
b = json.loads(open(f"gpurun_out/pdl/{c}_pdl{p}_r{r}.json").read().strip().splitlines()[-1])
print(c, "pdl", p, "rep", r, b["value"], b["ms_per_step"], b["phases_ms_per_step"], (b.get("roofline_step") or {}).get("achieved"))
PY
    done
  done
done
for rep in 1 2; do
  ASTRA_BENCH_PHASE_DUMP=1 timeout 400 python bench.py --config c3 > gpurun_out/pdl/c3_cpu_r$rep.json 2> gpurun_out/pdl/c3_cpu_r$rep.err
  python - $rep <<'PY'
import json, sys
r = sys.argv[1]
b = json.loads(open(f"gpurun_out/pdl/c3_cpu_r{r}.json").read().strip().splitlines()[-1])
err = open(f"gpurun_out/pdl/c3_cpu_r{r}.err").read().splitlines()
big = [l for l in err if l.startswith("step") and any(float(x) > 0.3 for x in l.split("[")[1].rstrip("]").split(","))]
print("c3 with cpu baseline rep", r, b["value"], b["ms_per_step"], b["phases_ms_per_step"], "stalled:", len(big), big[:4])
PY
done
