#!/bin/bash
mkdir -p gpurun_out/c3s
for rep in 1 2 3; do
  for cb in 0 1; do
    ASTRA_BENCH_PHASE_DUMP=1 timeout 400 python bench.py --config c3 $( [ $cb = 0 ] && echo --no-cpu-baseline ) > gpurun_out/c3s/c3_cb${cb}_r$rep.json 2> gpurun_out/c3s/c3_cb${cb}_r$rep.err
    python - $cb $rep <<'PY'
import json, sys
cb, r = sys.argv[1:]
f = f"gpurun_out/c3s/c3_cb{cb}_r{r}"
b = json.loads(open(f + ".json").read().strip().splitlines()[-1])
err = open(f + ".err").read().splitlines()
big = [l for l in err if l.startswith("step") and any(float(x) > 0.3 for x in l.split("[")[1].rstrip("]").split(","))]
gaps = [l for l in err if l.startswith("largest host gaps")]
print("c3 cpu_baseline", cb, "rep", r, b["value"], b["ms_per_step"], b["phases_ms_per_step"]["sample"], "stalled:", len(big), big[:2], gaps)
PY
  done
done
