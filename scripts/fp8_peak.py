"""Measured dense e4m3 tensor peak on this B200 (cuBLASLt via torch._scaled_mm,
8192^3, best of 10 CUDA-event timings after warm-up) -> profiles/fp8_peak.json.
MEASURED_PEAKS.json (driver-written) has no fp8 figure; this is the
denominator bench.py uses for the e4m3 refresh GEMM."""
import json
import os
import sys

import torch

n = 8192
a = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn)
b = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn).t()  # column-major B for cuBLASLt
one = torch.ones((), device="cuda")
for _ in range(5):
    torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
tf = 2 * n ** 3 / (best / 1e3) / 1e12
# bf16 burst the same way, for the ratio
x = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    x @ x
torch.cuda.synchronize()
bb = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x @ x
    e1.record()
    torch.cuda.synchronize()
    bb = min(bb, e0.elapsed_time(e1))
tb = 2 * n ** 3 / (bb / 1e3) / 1e12
out = {"fp8_e4m3_tflops": round(tf, 1), "bf16_tflops_same_run": round(tb, 1), "ratio": round(tf / tb, 3),
       "how": "torch._scaled_mm e4m3 8192^3 (cuBLASLt), best of 10 CUDA-event timings; bf16 torch.matmul 8192^3 likewise",
       "gpu": torch.cuda.get_device_name(0)}
print(json.dumps(out))
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "profiles", "fp8_peak.json")
json.dump(out, open(path, "w"), indent=1)
