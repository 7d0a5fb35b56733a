"""Step microbenchmark at the bench shape (L=1.3M, d=768, B=1024, S=584): ms per
minibatch of Philox slates + fused loss/update, and its HBM roofline."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_20156_b200.engine import ClassifierEngine  # noqa: E402

import os  # noqa: E402

L, d, B, k_p, k_h, k_r = 1_305_265, 768, 1024, 8, 64, 512
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
# ASTRA_BENCH_STEP_ADAM=1: bf16 W + Adam (the C5 shard's optimizer configuration)
adam = os.environ.get("ASTRA_BENCH_STEP_ADAM") == "1"
eng = ClassifierEngine(L, d, k_p=k_p, k_h=k_h, k_r=k_r, seed=0, w_dtype=torch.bfloat16 if adam else torch.float32,
                       optimizer="adam" if adam else "sgd")
g = torch.Generator(device="cuda")
g.manual_seed(1)
mbs = []
for t in range(4):
    rows = torch.arange(t * B, (t + 1) * B, device="cuda", dtype=torch.int64)
    pos = torch.randint(0, L, (B, 38), device="cuda", generator=g).sort(1).values.to(torch.int32)
    ip = torch.arange(0, B * 38 + 1, 38, device="cuda", dtype=torch.int64)
    hard = torch.randint(0, L, (B, k_h), device="cuda", generator=g).to(torch.int32)
    emb = torch.randn((B, d), device="cuda", generator=g)
    mbs.append((rows, ip, pos.reshape(-1).contiguous(), hard, emb))


# ASTRA_BENCH_STEP_GEMM=1: before every 9th minibatch, a C4-size refresh (the
# bench's power / cache environment for the step kernels); the refresh itself
# is outside the kernel timings reported for the step
gemm_env = os.environ.get("ASTRA_BENCH_STEP_GEMM") == "1"
if gemm_env:
    from paper_2409_20156_b200 import ops  # noqa: E402

    Wr = eng.W if eng.W.dtype == torch.float32 else eng.W.float()
    Wrb = ops.f32_to_bf16(Wr)
    Eq = torch.randn((9216, d), device="cuda", generator=g)
    pq = torch.randint(0, L, (9216, 38), device="cuda", generator=g).sort(1).values.to(torch.int32).reshape(-1)
    iq = torch.arange(0, 9216 * 38 + 1, 38, device="cuda", dtype=torch.int64)


def one(i):
    rows, ip, pid, hard, emb = mbs[i % 4]
    sl = eng.sample(rows, ip, pid, hard, epoch=1, step=i)
    return eng.step(emb, sl, 0.05, 1e-4), sl


for i in range(3):
    one(i)
torch.cuda.synchronize()
from paper_2409_20156_b200 import _lib  # noqa: E402

_lib.kernel_timing_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time  # noqa: E402

e0.record()
h0 = time.perf_counter()
pos = []
for i in range(n):
    if gemm_env and i % 9 == 0:
        ops.refresh_topk(Eq, iq, pq, k_h, "bf16_rerank", labels_f32=Wr, labels_bf16=Wrb)
    a_ = torch.cuda.Event(enable_timing=True)
    b_ = torch.cuda.Event(enable_timing=True)
    a_.record()
    _, sl = one(i)
    b_.record()
    pos.append((i % 9, a_, b_))
h1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"host {1e3 * (h1 - h0) / n:.3f} ms/minibatch (python + launches, no sync)")
U = int(torch.unique(sl[0]).numel())
byts = U * d * (2 * 2 + 16 if adam else 8) + 2 * B * d * 4 + B * (k_p + k_h + k_r) * 5
print(f"step {ms:.3f} ms/minibatch  U={U}  {byts / ms / 1e6:.0f} GB/s algorithmic ({byts / 1e9:.2f} GB)")
kt = {k: _lib.kernel_timing(k) for k in ("step_single", "slot_forward", "label_update")}
print("kernels  " + "  ".join(f"{k} {ms / max(c, 1):.3f} ms" for k, (ms, c) in kt.items()))
if gemm_env:
    per = [[] for _ in range(9)]
    for p_, a_, b_ in pos:
        per[p_].append(a_.elapsed_time(b_))
    print("minibatch ms by position after the refresh: " + " ".join(f"{sum(v) / len(v):.3f}" for v in per if v))
