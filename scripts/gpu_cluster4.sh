#!/bin/bash
# 2-pair (4-CTA) refresh cluster: a guarded first run, parity tests, A/B in the bench, ncu of the threshold pass
set -u
mkdir -p gpurun_out
ASTRA_TC_CLUSTER=4 timeout 120 python -m pytest tests/test_gpu_refresh.py -m gpu -q -x --timeout 100 -p no:cacheprovider > gpurun_out/c4_first.log 2>&1; rc=$?
echo "first_rc=$rc" >> gpurun_out/c4_first.log
tail -3 gpurun_out/c4_first.log
if [ $rc -ne 0 ]; then exit 0; fi
ASTRA_TC_CLUSTER=4 timeout 600 python -m pytest tests/test_gpu_refresh_scale.py -m gpu -q --timeout 500 -p no:cacheprovider > gpurun_out/c4_scale.log 2>&1; echo "rc=$?" >> gpurun_out/c4_scale.log
tail -3 gpurun_out/c4_scale.log
for i in 1 2; do
  for cl in 2 4; do
    ASTRA_TC_CLUSTER=$cl timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cl$cl.json 2>/dev/null
    python -c "
import json; b=json.loads(open('gpurun_out/bench_cl$cl.json').read().strip().splitlines()[-1])
print('cl=$cl', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'gemm', b['roofline']['launch_ms'], b['roofline']['frac'], b['refresh_parity']['recall_at_k'], b['clocks']['sm_mhz'], 'fp8', b['alt_fp8_refresh']['roofline']['launch_ms'])"
  done
done
ASTRA_TC_CLUSTER=4 timeout 600 python bench.py --config c5shard --no-cpu-baseline --steps 6 > gpurun_out/bench_c5_cl4.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/bench_c5_cl4.json').read().strip().splitlines()[-1])
print('c5 cl=4', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'gemm', b['roofline']['launch_ms'], b['roofline']['frac'], b['clocks']['sm_mhz'])"
ASTRA_TC_CLUSTER=4 timeout 600 ncu --set full --clock-control none -k regex:"refresh_tc_kernel" -s 2 -c 1 \
  -o gpurun_out/prof_refresh_cl4 python scripts/bench_refresh_k.py 9216 96 > gpurun_out/ncu_cl4.log 2>&1
tail -2 gpurun_out/ncu_cl4.log
