"""The PyTorch-encoder boundary (encoder.py:140-158): the
fused classifier step as an autograd node. A torch encoder's gradients after
loss.backward() must equal the chain rule through the ORACLE's grad_emb, and
W / the loss must match the oracle (oracle/xcmix_port.slate_step,
trainer.py:366-394) within the fp32 tolerance (1e-5 relative)."""

import numpy as np
import pytest
import torch

from oracle import xcmix_port as port
from test_gpu_step import close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [128, 768])
def test_torch_encoder_gets_grad_emb(cuda_lib, d):
    from paper_2409_20156_b200.autograd import slate_loss
    from paper_2409_20156_b200.engine import ClassifierEngine

    L, B, F, k_p, k_h, k_r = 20_000, 48, 64, 4, 16, 64
    torch.manual_seed(0)
    eng = ClassifierEngine(L, d, k_p=k_p, k_h=k_h, k_r=k_r, seed=3)
    W0 = eng.W.detach().cpu().numpy().copy()
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    rows = torch.arange(B, dtype=torch.int64, device="cuda")
    pos = torch.randint(0, L, (B, 5), device="cuda", generator=g).sort(1).values.to(torch.int32)
    ip = torch.arange(0, B * 5 + 1, 5, device="cuda", dtype=torch.int64)
    hard = torch.randint(0, L, (B, k_h), device="cuda", generator=g).to(torch.int32)
    slates = eng.sample(rows, ip, pos.reshape(-1).contiguous(), hard, epoch=3, step=0)

    enc = torch.nn.Sequential(torch.nn.Linear(F, d), torch.nn.Tanh()).cuda()
    x = torch.randn((B, F), device="cuda", generator=g)
    emb = enc(x)
    loss = slate_loss(emb, eng, slates, 0.05, 1e-4)
    loss.backward()
    got = [p.grad.detach().cpu().numpy() for p in enc.parameters()]

    ids, y, origin, weights = (t.cpu().numpy() for t in slates)
    Wref = W0.copy()
    rl, rge, _, uids = port.slate_step(Wref, emb.detach().cpu().numpy(), None, ids.astype(np.int64), y, origin,
                                       weights, 0.05, 1e-4)
    assert abs(float(loss) - rl) <= 1e-5 * abs(rl)
    close(eng.W.detach().cpu().numpy()[uids], Wref[uids])
    enc.zero_grad()
    want = torch.autograd.grad(enc(x), list(enc.parameters()), grad_outputs=torch.from_numpy(rge).cuda())
    for a, b in zip(got, want):
        close(a, b.cpu().numpy())


def test_nonfinite_raises_and_leaves_w(cuda_lib):
    from paper_2409_20156_b200.autograd import slate_loss
    from paper_2409_20156_b200.engine import ClassifierEngine
    from paper_2409_20156_b200.errors import NumericalError

    L, d, B = 5000, 128, 8
    eng = ClassifierEngine(L, d, k_p=2, k_h=0, k_r=16, seed=1)
    W0 = eng.W.detach().clone()
    rows = torch.arange(B, dtype=torch.int64, device="cuda")
    ip = torch.arange(0, B + 1, dtype=torch.int64, device="cuda")
    pos = torch.arange(B, dtype=torch.int32, device="cuda")
    slates = eng.sample(rows, ip, pos, None, epoch=0, step=0)
    emb = torch.full((B, d), float("inf"), device="cuda", requires_grad=True)
    with pytest.raises(NumericalError):
        slate_loss(emb, eng, slates, 0.1, 0.0)
    assert torch.equal(eng.W, W0)
