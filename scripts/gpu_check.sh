#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the top kernels.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:refresh_tc_kernel -s 2 -c 1 \
    -o gpurun_out/prof_refresh_tc python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_tc.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"label_update_vec|slot_forward_vec|rerank_kernel|merge_warp" -s 8 -c 4 \
    -o gpurun_out/prof_step python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_step.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
