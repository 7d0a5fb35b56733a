#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_refresh.py -q -x 2>&1 | tail -4
echo "== k sweep"; timeout 300 python scripts/bench_refresh_k.py 9216 1 32 64 96 2>&1 | grep -v cuBLAS
echo "== rerank"; timeout 300 python scripts/bench_refresh.py 9216 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_refresh.csv python scripts/bench_refresh_k.py 9216 96 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/launches_refresh.csv 2>&1 | head -12
