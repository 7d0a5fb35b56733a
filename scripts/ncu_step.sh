#!/bin/bash
# Launch list + one ncu --set full capture of the step kernels at the bench shape.
mkdir -p gpurun_out
timeout 300 python scripts/bench_step.py 20
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python scripts/bench_step.py 3 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/launches_step.csv 2>&1 | head -14
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slot_forward|label_update_tma" -s 4 -c 2 \
  -o gpurun_out/prof_step_${TAG:-x} python scripts/bench_step.py 3 > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
