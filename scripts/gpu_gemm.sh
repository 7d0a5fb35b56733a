#!/bin/bash
# 3xTF32 GEMM: guarded first run, parity tests, full-loss tests, fullloss bench line
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm_f32.py -m gpu -q -x --timeout 250 -p no:cacheprovider -s > gpurun_out/pytest_gemm.log 2>&1; rc=$?
echo "rc=$rc" >> gpurun_out/pytest_gemm.log
grep -E "gemm_f32|passed|failed|Error|error" gpurun_out/pytest_gemm.log | head -20
if [ $rc -ne 0 ]; then tail -30 gpurun_out/pytest_gemm.log; exit 0; fi
timeout 600 python -m pytest tests/test_gpu_full_loss.py tests/test_full_loss_dropin.py -m gpu -q --timeout 500 -p no:cacheprovider > gpurun_out/pytest_fl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fl.log
tail -3 gpurun_out/pytest_fl.log
timeout 600 python bench.py --config fullloss --steps 10 > gpurun_out/bench_fullloss.json 2> gpurun_out/bench_fullloss.err
tail -1 gpurun_out/bench_fullloss.json
