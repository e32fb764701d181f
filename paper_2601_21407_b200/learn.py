"""Training plumbing either side of the HH layer: the
reference's loss functions (learn.py:80-107) with their gradient seeds, on
the device.

`mse_loss` / `cross_entropy_loss` keep the reference signatures and return
(loss, seed) -- seed = d(loss)/d(pred), what `backward_through_time` takes as
seed_v.  `mse` is the autograd form used with `HHLayer`: one reduction pass
forward and one elementwise pass backward (torch's `(V*V).mean()` spends
five full passes over V on the same loss).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as nat
from .errors import UsageError


def _dev(x):
    return D.to_dev(x, np.float64, D.require_cuda()) if not D.is_dev(x) else x


def mse_loss(pred, target):
    """Mean squared error and its seed 2 (pred - target) / size (learn.py:80-88).
    numpy in -> (float, numpy float64); device tensors in -> (0-dim tensor, tensor)."""
    on_dev = D.is_dev(pred)
    if tuple(np.shape(pred)) != tuple(np.shape(target)):
        raise UsageError("mse_loss shape mismatch")
    p, t = _dev(pred), _dev(target).to(_dev(pred).dtype)
    diff = p - t
    loss = torch.linalg.vector_norm(diff).square() / diff.numel()
    seed = diff * (2.0 / diff.numel())
    if on_dev:
        return loss, seed
    return float(loss.item()), seed.double().cpu().numpy()


def cross_entropy_loss(logits, target):
    """Softmax cross-entropy over the trailing axis, mean over rows, and its seed
    (softmax - onehot) / rows (learn.py:92-107)."""
    on_dev = D.is_dev(logits)
    z = _dev(logits)
    y = target if D.is_dev(target) else torch.as_tensor(np.asarray(target), device=z.device)
    y = y.long()
    n = y.shape[0]
    logp = torch.log_softmax(z, dim=-1)
    loss = -logp[torch.arange(n, device=z.device), y].mean()
    seed = logp.exp()
    seed[torch.arange(n, device=z.device), y] -= 1.0
    seed /= n
    if on_dev:
        return loss, seed
    return float(loss.item()), seed.double().cpu().numpy()


class _MSE(torch.autograd.Function):
    @staticmethod
    def forward(ctx, v, target):
        diff = v if target is None else v - target
        ctx.save_for_backward(diff)
        ctx.has_target = target is not None
        return torch.linalg.vector_norm(diff).square() / diff.numel()

    @staticmethod
    def backward(ctx, g):
        (diff,) = ctx.saved_tensors
        c = 2.0 / diff.numel()
        if diff.dtype == torch.float32 and diff.is_contiguous() and g.dtype == torch.float32:
            seed = torch.empty_like(diff)
            nat.check(nat.load().hhb_scale_f32(diff.numel(), diff.data_ptr(), g.contiguous().data_ptr(), c,
                                               seed.data_ptr(), D.stream()), "hhb_scale_f32")
        else:
            seed = diff * (g * c)
        return seed, (-seed if ctx.has_target else None)


def mse(v: torch.Tensor, target: torch.Tensor | None = None) -> torch.Tensor:
    """Differentiable MSE(v, target) (target None = 0) for autograd training
    loops; the gradient is the reference's seed (learn.py:86-88)."""
    if target is not None and target.shape != v.shape:
        raise UsageError("mse shape mismatch")
    return _MSE.apply(v, target)
