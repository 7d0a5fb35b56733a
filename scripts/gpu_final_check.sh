#!/bin/bash
# Final check of the tree: smoke, the full GPU suite, the C4 headline and the drop-in line.
mkdir -p gpurun_out/fc
timeout 300 python __graft_entry__.py --smoke > gpurun_out/fc/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/fc/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/fc/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/fc/pytest_gpu.log
tail -3 gpurun_out/fc/pytest_gpu.log; tail -2 gpurun_out/fc/smoke.log
timeout 900 python bench.py > gpurun_out/fc/bench_c4.json 2> gpurun_out/fc/bench_c4.err
timeout 900 python bench.py --config dropin --steps 5 > gpurun_out/fc/bench_dropin.json 2> gpurun_out/fc/bench_dropin.err
for f in bench_c4 bench_dropin; do tail -1 gpurun_out/fc/$f.json | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('$f', b['value'], b['ms_per_step'], (b.get('e2e') or {}).get('value'), b.get('classifier_path_ms_per_step'), b.get('host_encoder_ms_per_step'))"; done
