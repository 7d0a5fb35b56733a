"""Single bf16_rerank refresh at the bench chunk size (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_20156_b200 import ops  # noqa: E402

L, d, k, nq = 1_305_265, 768, 64, int(sys.argv[1]) if len(sys.argv) > 1 else 9216
mode = sys.argv[2] if len(sys.argv) > 2 else "bf16_rerank"
g = torch.Generator(device="cuda")
g.manual_seed(0)
W = (torch.rand((L, d), device="cuda", generator=g) * 2 - 1) / d ** 0.5
Wb = ops.f32_to_bf16(W)
E = torch.randn((nq, d), device="cuda", generator=g)
pid = torch.randint(0, L, (nq, 38), device="cuda", generator=g).sort(1).values.to(torch.int32).reshape(-1).contiguous()
ip = torch.arange(0, nq * 38 + 1, 38, device="cuda", dtype=torch.int64)
for _ in range(3):
    ops.refresh_topk(E, ip, pid, k, mode, labels_f32=W, labels_bf16=Wb)
torch.cuda.synchronize()
