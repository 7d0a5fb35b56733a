#!/bin/bash
# single pass: slot released right after the W row is in registers (base) vs after grad_emb (late)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_full_loss.py tests/test_gpu_gemm_f32.py -m gpu -q --timeout 500 -p no:cacheprovider > gpurun_out/pytest_er.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_er.log
tail -2 gpurun_out/pytest_er.log
for i in 1 2; do
for v in base late; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  echo "== $v $(timeout 300 python scripts/bench_step.py 30 | tail -1)"
done
done
for i in 1 2; do
for v in base late; do
  if [ $v = base ]; then unset ASTRA_LIB_VARIANT; else export ASTRA_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --no-alt-fp8 --steps 10 > gpurun_out/bench_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1])
print('$v', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'single', b['roofline_step']['kernels']['step_single']['launch_ms'], 'gemm', b['roofline']['launch_ms'])"
done
done
unset ASTRA_LIB_VARIANT
timeout 600 python bench.py --config fullloss --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('fullloss', b['value'], b['ms_per_step'])"
