"""Repeat tests/test_gpu_step.py::test_adam_matches_torch_sparse_adam N times
in one process and count failures (race hunting; ASTRA_PDL from the env)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import test_gpu_step as T  # noqa: E402
from paper_2409_20156_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
lib = _lib.load()
fails = 0
msgs = []
for i in range(n):
    try:
        T.test_adam_matches_torch_sparse_adam(lib)
    except AssertionError as e:
        fails += 1
        if len(msgs) < 3:
            msgs.append(str(e).splitlines()[0][:120])
print(f"ASTRA_PDL={os.environ.get('ASTRA_PDL', '1')} runs={n} failures={fails}", msgs)
