#!/bin/bash
# Profiles for profiles/: bench launch list, ncu --set full of the refresh GEMM
# pass (threshold mode) and of the two step kernels.
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
# the 2nd refresh call's passes are launches 3 (sample), 4 (threshold), 5 (verify) of refresh_tc_kernel
SKIP=4 TAG=threshold bash scripts/ncu_refresh.sh
TAG=tma bash scripts/ncu_step.sh
python scripts/ncu_summary.py gpurun_out/launches_bench.csv gpurun_out/prof_tc_threshold.ncu-rep gpurun_out/prof_step_tma.ncu-rep > gpurun_out/ncu_summary.txt 2>&1
tail -60 gpurun_out/ncu_summary.txt
