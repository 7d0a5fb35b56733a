#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_checkpoint.py tests/test_device_bank.py -m gpu -q --timeout 600 -p no:cacheprovider -rf > gpurun_out/step_tests.log 2>&1; echo "rc=$?" >> gpurun_out/step_tests.log
timeout 900 python bench.py --config c5shard --steps 10 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "rc=$?" >> gpurun_out/c5.err
ASTRA_BENCH_STEP_ADAM=1 timeout 300 python scripts/bench_step.py 30 > gpurun_out/step_adam.txt 2>&1
ASTRA_BENCH_STEP_ADAM=1 ASTRA_STEP_SINGLE_ADAM=1 timeout 300 python scripts/bench_step.py 30 > gpurun_out/step_adam_single.txt 2>&1
timeout 300 python scripts/bench_step.py 30 > gpurun_out/step_sgd.txt 2>&1
ASTRA_BENCH_STEP_ADAM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"label_update_tma|slot_forward_tma" -s 4 -c 2 \
  -o gpurun_out/prof_adam python scripts/bench_step.py 3 > gpurun_out/ncu_adam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_single" -s 3 -c 1 \
  -o gpurun_out/prof_single python scripts/bench_step.py 3 > gpurun_out/ncu_single.log 2>&1
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/step_tests.log; cat gpurun_out/c5.json | head -c 1500; tail -2 gpurun_out/c5.err; tail -2 gpurun_out/step_adam.txt gpurun_out/step_adam_single.txt gpurun_out/step_sgd.txt; tail -2 gpurun_out/ncu_adam.log gpurun_out/ncu_single.log
