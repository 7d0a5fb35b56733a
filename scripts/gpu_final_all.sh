#!/bin/bash
# Round-2 final evidence on one box: smoke, the full GPU suite, the bench lines, the profiles.
set -u
mkdir -p gpurun_out/final
timeout 300 python __graft_entry__.py --smoke > gpurun_out/final/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/final/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/final/pytest_gpu.log
tail -4 gpurun_out/final/pytest_gpu.log; tail -2 gpurun_out/final/smoke.log
bash scripts/gpu_bench_final.sh
bash scripts/gpu_profile_final.sh > /dev/null 2>&1
rm -f gpurun_out/final/*.ncu-rep
head -60 gpurun_out/final/ncu_summary.txt
