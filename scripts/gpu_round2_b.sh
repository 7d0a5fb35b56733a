#!/bin/bash
# bench (with CPU baseline + refresh parity), emulated N-GPU lines, the reference arm, the ties test
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_refresh_scale.py -m gpu -q -s -k forced --timeout 600 -p no:cacheprovider > gpurun_out/ties.log 2>&1; echo "rc=$?" >> gpurun_out/ties.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
for n in 2 4 8; do
  timeout 900 python bench.py --emulate $n --steps 10 > gpurun_out/emulate_$n.json 2> gpurun_out/emulate_$n.err; echo "rc=$?" >> gpurun_out/emulate_$n.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "rc=$?" >> gpurun_out/ref.err
tail -3 gpurun_out/ties.log; tail -2 gpurun_out/bench.err; tail -1 gpurun_out/emulate_8.err; cat gpurun_out/ref.json; tail -2 gpurun_out/ref.err
