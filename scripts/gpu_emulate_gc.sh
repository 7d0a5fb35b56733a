#!/bin/bash
# emulated N-GPU lines with the global candidate threshold (default) and without (N = 8 A/B), same box
set -u
mkdir -p gpurun_out/emu
for n in 2 4 8; do
  timeout 900 python bench.py --emulate $n --steps 6 > gpurun_out/emu/emulate_${n}gpu.json 2>gpurun_out/emu/emulate_${n}gpu.err
  python -c "
import json; b=json.loads(open('gpurun_out/emu/emulate_${n}gpu.json').read().strip().splitlines()[-1])
print('N=$n', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'gemm', b['roofline']['launch_ms'])"
done
timeout 900 python bench.py --emulate 8 --emulate-shard-candidates --steps 6 > gpurun_out/emu/emulate_8gpu_shardcand.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/emu/emulate_8gpu_shardcand.json').read().strip().splitlines()[-1])
print('N=8 shard candidates', b['value'], b['ms_per_step'], b['phases_ms_per_step'], 'gemm', b['roofline']['launch_ms'])"
tail -3 gpurun_out/emu/emulate_8gpu.err
