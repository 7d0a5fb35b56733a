#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_importance.py tests/test_dropin_train_golden.py tests/test_device_bank.py -m gpu -q -s --timeout 600 -p no:cacheprovider -rf > gpurun_out/imp.log 2>&1; echo "rc=$?" >> gpurun_out/imp.log
timeout 900 python bench.py --config c5shard --steps 10 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "rc=$?" >> gpurun_out/c5.err
# the reference's own acceptance criterion 8 WITHOUT the drop-in (is its timing bar met on this host at all?)
cd baseline/_ref_tests && PYTHONPATH=../_ref timeout 900 python -m pytest test_acceptance.py -q -p no:cacheprovider -k "criterion_08" > ../../gpurun_out/ref_c8.log 2>&1; cd ../..
timeout 1200 python -m pytest tests/test_dropin_cuda.py -m gpu -q --timeout 1100 -p no:cacheprovider -rf > gpurun_out/dropin_cuda.log 2>&1; echo "rc=$?" >> gpurun_out/dropin_cuda.log
tail -4 gpurun_out/imp.log; cat gpurun_out/c5.json; tail -2 gpurun_out/c5.err; tail -3 gpurun_out/ref_c8.log; tail -3 gpurun_out/dropin_cuda.log
