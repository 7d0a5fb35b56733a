#!/bin/bash
# C3 host-stall check after the event pool / pre-created timing events, PDL on and off.
mkdir -p gpurun_out/c3s2
for rep in 1 2 3 4 5; do
  for pdl in 1; do
    ASTRA_PDL=$pdl ASTRA_BENCH_PHASE_DUMP=1 timeout 400 python bench.py --config c3 --no-cpu-baseline > gpurun_out/c3s2/c3_pdl${pdl}_r$rep.json 2> gpurun_out/c3s2/c3_pdl${pdl}_r$rep.err
    python - $pdl $rep <<'PY'
import json, sys
p, r = sys.argv[1:]
f = f"gpurun_out/c3s2/c3_pdl{p}_r{r}"
b = json.loads(open(f + ".json").read().strip().splitlines()[-1])
err = open(f + ".err").read().splitlines()
big = [l for l in err if l.startswith("step") and any(float(x) > 0.3 for x in l.split("[")[1].rstrip("]").split(","))]
gaps = [l for l in err if l.startswith("largest host gaps")]
print("c3 pdl", p, "rep", r, b["value"], b["ms_per_step"], b["phases_ms_per_step"], "stalled:", len(big), big[:2], gaps)
PY
  done
done
