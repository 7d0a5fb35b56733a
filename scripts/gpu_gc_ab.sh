#!/bin/bash
# GC on (collections logged) vs off (default) for the short-step lines.
mkdir -p gpurun_out/gc
for rep in 1 2 3; do
  for gcon in 1 0; do
    for c in c2 c3; do
      if [ $gcon = 1 ]; then export ASTRA_BENCH_GC=1; else unset ASTRA_BENCH_GC; fi
      ASTRA_BENCH_PHASE_DUMP=1 timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/gc/${c}_gc${gcon}_r$rep.json 2> gpurun_out/gc/${c}_gc${gcon}_r$rep.err
      python - $c $gcon $rep <<'PY'
import json, sys
c, g, rep = sys.argv[1:]
f = f"gpurun_out/gc/{c}_gc{g}_r{rep}"
b = json.loads(open(f + ".json").read().strip().splitlines()[-1])
err = open(f + ".err").read().splitlines()
big = [l for l in err if l.startswith("step") and any(float(x) > 0.3 for x in l.split("[")[1].rstrip("]").split(","))]
gcs = [l for l in err if l.startswith("gc gen2")]
print(c, "gc", g, "rep", rep, b["value"], b["ms_per_step"], b["phases_ms_per_step"]["sample"], "stalled:", len(big), big[:2], "gen2:", gcs[-4:])
PY
    done
  done
done
