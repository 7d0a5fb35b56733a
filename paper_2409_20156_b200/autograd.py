"""The encoder boundary for a PyTorch encoder.

The reference's encoder is NumPy: `_batch_forward_backward` (trainer.py:336-395)
computes grad_emb in the classifier half and hands it to
`encoder_backward_batch` (encoder.py:140-158), which raises on a non-finite
grad_emb before touching anything (encoder.py:145-146). The paper's encoder
(DistilBERT) is a PyTorch module; for it the classifier step is one autograd
node:

    emb = encoder(x)                                  # [B, d] on the GPU
    loss = slate_loss(emb, engine, slates, lr, wd)    # fused step: loss with the
                                                      # current W, W updated in place
    loss.backward()                                   # encoder grads from grad_emb

forward runs `ClassifierEngine.step` (astra_slate_step: scores, BCE terms,
factors, grad_emb, the sparse SGD/Adam row update — the same call as the
reference's classifier half), backward returns grad_emb (scaled by the
incoming gradient) to the encoder's graph without leaving the device. Dropout
is the caller's (apply it to `emb` before the call; autograd carries the keep
mask, which is what the reference's `keep` scaling of grad_emb does).
"""

from __future__ import annotations

import torch

from .errors import NumericalError


class SlateLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, emb, engine, slates, lr, weight_decay, check):
        loss, grad_emb, status = engine.step(emb.detach().contiguous(), slates, lr, weight_decay)
        if check:
            st = status.cpu().tolist()
            if st[0] or st[1]:
                # classifiers.py:79-80 / encoder.py:145-146: nothing written, raise
                raise NumericalError("non-finite classifier gradient")
        ctx.save_for_backward(grad_emb)
        return loss.reshape(()).to(torch.float64)

    @staticmethod
    def backward(ctx, grad_out):
        (grad_emb,) = ctx.saved_tensors
        g = grad_emb if grad_out is None else grad_emb * grad_out.to(grad_emb.dtype)
        return g, None, None, None, None, None


def slate_loss(emb: torch.Tensor, engine, slates, lr: float, weight_decay: float = 0.0,
               check: bool = True) -> torch.Tensor:
    """Summed sampled-BCE loss of one minibatch (fp64 scalar) as an autograd
    node over `emb`; applies the classifier update on `engine` as a side
    effect (trainer.py:382-394). check=True synchronises once to raise
    NumericalError on a non-finite gradient (W is then untouched)."""
    return SlateLoss.apply(emb, engine, slates, lr, weight_decay, check)
