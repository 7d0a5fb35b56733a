#!/bin/bash
# Final round-2 bench lines (one box): C4 headline (with the CPU reference beside it), the reference arm,
# C1/C2/C3, C5 shard, drop-in, full-loss arm, emulated N = 2/4/8.
set -u
O=gpurun_out/final_bench
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for c in c1 c2 c3 c5shard dropin fullloss; do
  timeout 900 python bench.py --config $c $( [ $c = dropin ] && echo "--steps 5" ) > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --w-init clustered --no-cpu-baseline --steps 10 > $O/bench_c4_clustered.json 2> $O/bench_c4_clustered.err
for n in 2 4 8; do
  timeout 900 python bench.py --emulate $n --steps 6 > $O/emulate_${n}gpu.json 2> $O/emulate_${n}gpu.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/final_bench/*.json")):
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], b.get("value"), b.get("unit"), b.get("ms_per_step"), (b.get("e2e") or {}).get("value"),
              (b.get("roofline") or {}).get("frac"), (b.get("cpu_baseline") or {}).get("value"), (b.get("clocks") or {}).get("sm_mhz"))
    except Exception as e:
        print(f, "ERR", e)
PY
