#!/bin/bash
# Profiles for profiles/: bench launch list, ncu --set full of the refresh GEMM
# pass (threshold mode), of the single-pass step kernel and of the two-kernel
# step schedule. Summaries are written on the box (gpurun_out/ncu_summary.txt);
# KEEP_REPS=1 keeps the .ncu-rep files (large).
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
# the 2nd refresh call's passes are launches 3 (sample), 4 (threshold), 5 (verify) of refresh_tc_kernel
SKIP=4 TAG=threshold bash scripts/ncu_refresh.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_single" -s 3 -c 1 \
  -o gpurun_out/prof_single_final python scripts/bench_step.py 3 > gpurun_out/ncu_single.log 2>&1
ASTRA_STEP_SINGLE=0 TAG=tma bash scripts/ncu_step.sh
python scripts/ncu_summary.py gpurun_out/launches_bench.csv gpurun_out/prof_tc_threshold.ncu-rep \
  gpurun_out/prof_single_final.ncu-rep gpurun_out/prof_step_tma.ncu-rep > gpurun_out/ncu_summary.txt 2>&1
for r in tc_threshold single_final step_tma; do
  ncu -i gpurun_out/prof_$r.ncu-rep --page details --csv > gpurun_out/details_$r.csv 2>/dev/null
done
if [ "${KEEP_REPS:-0}" != 1 ]; then rm -f gpurun_out/*.ncu-rep; fi
tail -80 gpurun_out/ncu_summary.txt
