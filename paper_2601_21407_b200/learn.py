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


# ---------------------------------------------------------------------------
# synaptic filtering, metric, optimizer (learn.py:33-156)
# ---------------------------------------------------------------------------

import math
from dataclasses import dataclass, field

from .errors import ConfigurationError


@dataclass(frozen=True)
class PSPKernel:
    """Causal exponential-decay kernel, taps normalised to unit sum (learn.py:33-49)."""

    tau_decay: float
    length: int
    dt: float = 0.1

    def __post_init__(self):
        if self.tau_decay <= 0:
            raise ConfigurationError("tau_decay must be > 0")
        if self.length < 1:
            raise ConfigurationError("kernel length must be >= 1")

    @property
    def taps(self) -> np.ndarray:
        w = np.exp(-np.arange(self.length) * self.dt / self.tau_decay)
        return w / w.sum()


def psp_filter(spikes, kernel: PSPKernel):
    """Causal convolution along the leading (time) axis (learn.py:52-55), on the
    device (hhb_psp_filter, scipy.signal.lfilter's operation order).  numpy in ->
    float64 numpy out; CUDA tensors in -> tensors of their dtype out."""
    on_dev = D.is_dev(spikes)
    dev = spikes.device if on_dev else D.require_cuda()
    dtype = (np.float32 if spikes.dtype == torch.float32 else np.float64) if on_dev else np.float64
    x = D.to_dev(spikes, dtype, dev).contiguous()
    shape = tuple(x.shape)
    T = shape[0] if shape else 0
    cols = int(np.prod(shape[1:], dtype=np.int64)) if len(shape) > 1 else 1
    taps = torch.tensor(kernel.taps, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    nat.check(nat.load().hhb_psp_filter(D.code(x.dtype), T, cols, int(taps.numel()), taps.data_ptr(), x.data_ptr(),
                                        y.data_ptr(), D.stream()), "hhb_psp_filter")
    return y if on_dev else y.cpu().numpy()


def smape(pred, truth) -> float:
    """Symmetric mean absolute percentage error in [0, 100] (learn.py:62-77)."""
    p = _dev(pred).double().reshape(-1)
    t = _dev(truth).double().reshape(-1)
    if p.numel() == 0:
        raise UsageError("smape requires non-empty input")
    if p.shape != t.shape:
        raise UsageError("smape requires equal-length inputs")
    num = (p - t).abs()
    den = p.abs() + t.abs()
    terms = torch.where(den > 0, num / torch.where(den > 0, den, torch.ones_like(den)), torch.zeros_like(num))
    return float(100.0 * terms.mean().item())


@dataclass
class AdamState:
    """Bias-corrected Adam with per-parameter moment buffers (learn.py:114-124)."""

    lr: float = 5e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)


def adam_step(params: dict, grads: dict, state: AdamState, lr: float | None = None) -> dict:
    """One Adam update (learn.py:127-146) in the reference's operation order,
    float64 on the device; numpy params in -> numpy out, tensors -> tensors."""
    state.step += 1
    t = state.step
    lr = state.lr if lr is None else lr
    out = {}
    b1, b2 = state.beta1, state.beta2
    c1, c2 = 1 - b1 ** t, 1 - b2 ** t
    for name, p in params.items():
        on_dev = D.is_dev(p)
        g = _dev(grads[name]).double()
        m = state.m.get(name)
        if m is None:
            m = torch.zeros_like(g)
            state.m[name] = m
            state.v[name] = torch.zeros_like(g)
        v = state.v[name]
        m.copy_(b1 * m + (1 - b1) * g)
        v.copy_(b2 * v + (1 - b2) * g * g)
        m_hat = m / c1
        v_hat = v / c2
        new = _dev(p).double() - lr * m_hat / (torch.sqrt(v_hat) + state.eps)
        out[name] = new if on_dev else new.cpu().numpy()
    return out


def cosine_lr(base_lr: float, epoch: int, total_epochs: int) -> float:
    """Cosine annealing from base_lr to 0 over the run (learn.py:149-151)."""
    return base_lr * 0.5 * (1.0 + math.cos(math.pi * epoch / max(total_epochs, 1)))
