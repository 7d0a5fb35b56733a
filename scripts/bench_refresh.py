"""Refresh microbenchmark: q/s and TFLOP/s of the bf16 tcgen05 refresh vs batch size."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_20156_b200 import ops  # noqa: E402

L, d, k = 1_305_265, 768, 64
g = torch.Generator(device="cuda")
g.manual_seed(0)
W = (torch.rand((L, d), device="cuda", generator=g) * 2 - 1) / d ** 0.5
Wb = ops.f32_to_bf16(W)
res = {}
for nq in [int(x) for x in (sys.argv[1:] or ["1024", "4096", "9472", "18944"])]:
    E = torch.randn((nq, d), device="cuda", generator=g)
    pos = torch.randint(0, L, (nq, 38), device="cuda", generator=g).sort(1).values.to(torch.int32)
    ip = torch.arange(0, nq * 38 + 1, 38, device="cuda", dtype=torch.int64)
    pid = pos.reshape(-1).contiguous()
    for mode in ("bf16", "bf16_rerank"):
        for _ in range(2):
            ops.refresh_topk(E, ip, pid, k, mode, labels_f32=W, labels_bf16=Wb)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 5
        e0.record()
        for _ in range(n):
            ops.refresh_topk(E, ip, pid, k, mode, labels_f32=W, labels_bf16=Wb)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        tf = 2 * L * d * nq / (ms / 1e3) / 1e12
        res[f"{mode}_{nq}"] = {"ms": round(ms, 3), "qps": round(nq / ms * 1e3), "tflops": round(tf, 1)}
        print(mode, nq, res[f"{mode}_{nq}"], flush=True)
json.dump(res, open("gpurun_out/bench_refresh.json", "w"), indent=1)
