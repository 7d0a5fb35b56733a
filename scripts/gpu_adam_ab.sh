#!/bin/bash
# A/B of the bf16 + Adam update variants (IEEE vs MUFU sqrt/rcp; 3 vs 4 CTAs/SM),
# C4-shape microbenchmark and the C5 shard bench line; ncu source capture of step_single.
set -u
mkdir -p gpurun_out
bash scripts/ab_step_adam.sh base fast fast4 > gpurun_out/ab_adam_micro.txt 2>&1
for v in base fast fast4; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  timeout 900 python bench.py --config c5shard --no-cpu-baseline --steps 6 > gpurun_out/c5_$v.json 2> gpurun_out/c5_$v.err
  python -c "
import json; b=json.loads(open('gpurun_out/c5_$v.json').read().strip().splitlines()[-1])
print('$v', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline_step'].get('label_update_launch_ms'), b['clocks']['sm_mhz'])" >> gpurun_out/ab_adam_c5.txt 2>&1
done
unset ASTRA_LIB_VARIANT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_single" -s 3 -c 1 \
  -o gpurun_out/prof_single_src python scripts/bench_step.py 3 > gpurun_out/ncu_single.log 2>&1
cat gpurun_out/ab_adam_micro.txt gpurun_out/ab_adam_c5.txt
