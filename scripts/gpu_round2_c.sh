#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
for n in 2 8; do
  ASTRA_PROFILE_REFRESH=1 timeout 600 python bench.py --emulate $n --steps 4 > gpurun_out/emulate_prof_$n.json 2> gpurun_out/emulate_prof_$n.err
done
for n in 2 4 8; do
  timeout 900 python bench.py --emulate $n --steps 10 > gpurun_out/emulate_$n.json 2> gpurun_out/emulate_$n.err; echo "rc=$?" >> gpurun_out/emulate_$n.err
done
tail -15 gpurun_out/pytest_gpu.log; grep "refresh stages" gpurun_out/emulate_prof_8.err | tail -2
