#!/bin/bash
# fullloss bench line (tf32 GEMM roofline), C5 shard: two-kernel Adam (default) vs single pass Adam (same box),
# ncu --set full of one gemm_f32 launch
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --config fullloss --steps 10 > gpurun_out/bench_fullloss.json 2> gpurun_out/bench_fullloss.err
tail -1 gpurun_out/bench_fullloss.json
for i in 1 2; do
for s in 0 1; do
  ASTRA_STEP_SINGLE_ADAM=$s timeout 900 python bench.py --config c5shard --no-cpu-baseline --steps 6 > gpurun_out/c5_single$s.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/c5_single$s.json').read().strip().splitlines()[-1])
print('single_adam=$s', b['value'], b['ms_per_step'], b['phases_ms_per_step'], b['roofline_step'].get('label_update_launch_ms'), b['clocks']['sm_mhz'])"
done
done
timeout 600 ncu --set full --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/prof_gemm_f32 python bench.py --config fullloss --steps 2 --warmup 1 > gpurun_out/ncu_gemm.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_gemm_f32.ncu-rep > gpurun_out/ncu_gemm_summary.txt 2>&1; cat gpurun_out/ncu_gemm_summary.txt
