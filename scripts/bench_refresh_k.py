"""Refresh time vs k (epilogue cost) and vs a cuBLAS bf16 GEMM of the same flops."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_20156_b200 import ops  # noqa: E402

L, d, nq = 1_305_265, 768, int(sys.argv[1]) if len(sys.argv) > 1 else 9216
g = torch.Generator(device="cuda")
g.manual_seed(0)
W = (torch.rand((L, d), device="cuda", generator=g) * 2 - 1) / d ** 0.5
Wb = ops.f32_to_bf16(W)
E = torch.randn((nq, d), device="cuda", generator=g)
pid = torch.randint(0, L, (nq, 38), device="cuda", generator=g).sort(1).values.to(torch.int32).reshape(-1).contiguous()
ip = torch.arange(0, nq * 38 + 1, 38, device="cuda", dtype=torch.int64)


def timeit(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for k in [int(x) for x in (sys.argv[2:] or ["1", "8", "32", "64", "96", "128"])]:
    ms = timeit(lambda: ops.refresh_topk(E, ip, pid, k, "bf16", labels_f32=W, labels_bf16=Wb))
    print(f"bf16 k={k}: {ms:.3f} ms  {2 * L * d * nq / ms / 1e9:.1f} TFLOP/s", flush=True)
# cuBLAS reference: same flops in 10 chunks of L/10 (bf16 out)
Eb = E.to(torch.bfloat16)
ch = (L + 9) // 10
outs = torch.empty((nq, ch), dtype=torch.bfloat16, device="cuda")


def cublas():
    for i in range(10):
        torch.matmul(Eb, Wb[i * ch : (i + 1) * ch].T, out=outs[:, : min(ch, L - i * ch)])


ms = timeit(cublas, 3)
print(f"cuBLAS bf16 (scores materialised): {ms:.3f} ms  {2 * L * d * nq / ms / 1e9:.1f} TFLOP/s", flush=True)
