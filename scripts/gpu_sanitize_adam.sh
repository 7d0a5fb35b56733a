#!/bin/bash
# compute-sanitizer on the Adam/SparseAdam parity test (the intermittent failure), and a loop of the test
set -u
mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -m gpu -q -k "adam_matches" -p no:cacheprovider > gpurun_out/san/initcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san/initcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_step.py -m gpu -q -k "adam_matches" -p no:cacheprovider > gpurun_out/san/racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san/racecheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -m gpu -q -k "adam_matches" -p no:cacheprovider > gpurun_out/san/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san/memcheck.log
tail -15 gpurun_out/san/initcheck.log; tail -8 gpurun_out/san/racecheck.log; tail -8 gpurun_out/san/memcheck.log
cat > /tmp/loop_adam.py <<'PY'
import sys, subprocess
fails = 0
for i in range(12):
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_step.py", "-m", "gpu", "-q", "-k", "adam_matches or bitexact or fuzz", "-p", "no:cacheprovider"], capture_output=True, text=True)
    ok = r.returncode == 0
    fails += not ok
    print(i, "ok" if ok else "FAIL", r.stdout.strip().splitlines()[-1])
print("fails", fails)
PY
timeout 1200 python /tmp/loop_adam.py
