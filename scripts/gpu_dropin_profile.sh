#!/bin/bash
# The drop-in line, then a host profile of its timed steps (cProfile, tottime).
mkdir -p gpurun_out/dropin
timeout 600 python bench.py --config dropin --steps 5 > gpurun_out/dropin/bench_dropin.json 2> gpurun_out/dropin/bench_dropin.err
tail -1 gpurun_out/dropin/bench_dropin.json | python -c "import json,sys; b=json.loads(sys.stdin.read()); print(b['value'], b['ms_per_step'], b['host_encoder_ms_per_step'], b['classifier_path_ms_per_step'])"
ASTRA_BENCH_PROFILE=1 timeout 600 python bench.py --config dropin --steps 5 > /dev/null 2> gpurun_out/dropin/prof.txt
grep -A40 "Ordered by" gpurun_out/dropin/prof.txt | head -45
