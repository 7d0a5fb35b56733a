#!/bin/bash
# Final round-2 evidence: launch list of the C4 bench; ncu --set full of the refresh threshold pass
# (bf16, bench shape), step_single in the bench (cache state of the real step) and in the microbenchmark,
# the bf16+Adam single pass, the 3xTF32 GEMM; summaries + raw details.
set -u
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-alt-fp8 > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:refresh_tc_kernel -s 4 -c 1 \
  -o $O/prof_threshold python scripts/bench_refresh_k.py 9216 96 > $O/ncu_threshold.log 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:step_single -s 40 -c 1 \
  -o $O/prof_single_inbench python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-alt-fp8 > $O/ncu_single_inbench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_single -s 3 -c 1 \
  -o $O/prof_single_micro python scripts/bench_step.py 3 > $O/ncu_single_micro.log 2>&1
ASTRA_BENCH_STEP_ADAM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_single -s 3 -c 1 \
  -o $O/prof_single_adam python scripts/bench_step.py 3 > $O/ncu_single_adam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
  -o $O/prof_gemm_f32 python bench.py --config fullloss --steps 3 --warmup 3 > $O/ncu_gemm.log 2>&1
python scripts/ncu_summary.py $O/launches_bench.csv $O/prof_threshold.ncu-rep $O/prof_single_inbench.ncu-rep \
  $O/prof_single_micro.ncu-rep $O/prof_single_adam.ncu-rep $O/prof_gemm_f32.ncu-rep > $O/ncu_summary.txt 2>&1
for r in threshold single_inbench single_micro single_adam gemm_f32; do
  python scripts/ncu_sass_hot.py $O/prof_$r.ncu-rep 20 > $O/sass_hot_$r.txt 2>&1
done
tail -100 $O/ncu_summary.txt
