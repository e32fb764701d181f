"""Drop-in for `hhengine.learn`: the training plumbing either side
of the HH hot path, on the device.

* losses with their gradient seeds (learn.py:80-107): `mse_loss`,
  `cross_entropy_loss` return (loss, seed), seed = d(loss)/d(pred), what
  `backward_through_time` takes as seed_v; `mse` is the autograd form for
  `HHLayer` outputs (one reduction forward, one `hhb_scale_f32` pass back);
* `PSPKernel` / `psp_filter` (causal FIR, CUDA, lfilter's operation order),
  `smape`, `AdamState` / `adam_step`, `cosine_lr` (learn.py:33-151);
* trace segmentation and dataset split, the dense layer, the teacher-student
  `ReadoutModel` (readout GEMV kernels around the HH forward/BPTT kernels),
  `make_teacher_student_task` / `make_student` / `fit` / `evaluate_smape`, and
  the ndjson dataset / csv history files (learn.py:158-415).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from . import _native as nat
from .errors import ConfigurationError, TrainingDivergedError, UsageError


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


def _smape_dev(p: torch.Tensor, t: torch.Tensor) -> torch.Tensor:
    p, t = p.double().reshape(-1), t.double().reshape(-1)
    num = (p - t).abs()
    den = p.abs() + t.abs()
    terms = torch.where(den > 0, num / torch.where(den > 0, den, torch.ones_like(den)), torch.zeros_like(num))
    return 100.0 * terms.mean()


def smape(pred, truth) -> float:
    """Symmetric mean absolute percentage error in [0, 100] (learn.py:62-77)."""
    p = _dev(pred).double().reshape(-1)
    t = _dev(truth).double().reshape(-1)
    if p.numel() == 0:
        raise UsageError("smape requires non-empty input")
    if p.shape != t.shape:
        raise UsageError("smape requires equal-length inputs")
    return float(_smape_dev(p, t).item())


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


# ---------------------------------------------------------------------------
# trace segmentation and dataset split (learn.py:158-196)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SegmentationScheme:
    """pad_len warm-up steps followed by out_len supervised steps per sample;
    consecutive supervised windows tile the trace (learn.py:158-170)."""

    pad_len: int
    out_len: int

    def __post_init__(self):
        if self.pad_len < 0 or self.out_len <= 0:
            raise ConfigurationError("invalid segmentation scheme")


def segment_traces(input_trace, output_trace, scheme: SegmentationScheme):
    """[(input[lo:lo+pad+out], output[lo+pad:lo+pad+out]) for lo = k*out_len]
    (learn.py:173-189); views of the caller's arrays, as the reference."""
    x = np.asarray(input_trace)
    y = np.asarray(output_trace)
    if x.shape[0] != y.shape[0]:
        raise UsageError("input and output traces must share length")
    count = max((x.shape[0] - scheme.pad_len) // scheme.out_len, 0)
    width = scheme.pad_len + scheme.out_len
    return [(x[k * scheme.out_len:k * scheme.out_len + width],
             y[k * scheme.out_len + scheme.pad_len:k * scheme.out_len + width]) for k in range(count)]


def split_dataset(n_samples: int, rng: np.random.Generator, ratio=(3, 1)):
    """Shuffled (train, test) index split, floor on the train side (learn.py:192-196)."""
    order = rng.permutation(n_samples)
    cut = n_samples * ratio[0] // (ratio[0] + ratio[1])
    return order[:cut], order[cut:]


# ---------------------------------------------------------------------------
# dense layer and the teacher-student readout model (learn.py:203-274)
# ---------------------------------------------------------------------------

@dataclass
class DenseLayer:
    """y = x @ W.T + b over the trailing axis (learn.py:203-216).  numpy in ->
    numpy out (computed on the device, float64 as the reference); CUDA tensors
    in -> tensors out, float32 ones through the tcgen05 GEMM (bf16x3)."""

    weights: object   # (out, in)
    bias: object      # (out,)

    def __call__(self, x):
        on_dev = D.is_dev(x)
        xd = _dev(x)
        if xd.dtype == torch.float32:
            # float32 device operands: the tcgen05 GEMM in its fp32-class bf16x3
            # form (x and W split into bf16 hi + lo, three tensor-core products)
            from .layer import _stream, _workspace, gemm, split3_padded
            from . import _native as nat
            k = xd.shape[-1]
            x2 = xd.reshape(-1, k).contiguous()
            wa, kp = split3_padded(_dev(self.weights).float().reshape(-1, k).contiguous(), 1)   # [W_hi|W_hi|W_lo]
            b32 = _dev(self.bias).float().contiguous()
            M, N = x2.shape[0], wa.shape[0]
            if M >= 512 and k % 4 == 0 and N % 4 == 0:      # (CTA-pair tiles, 16-byte row pitches)
                # x split into hi / lo on chip inside the GEMM (hhb_gemm_f32a)
                lib = nat.load()
                y = torch.empty((M, N), dtype=torch.float32, device=x2.device)
                ws_n = int(lib.hhb_gemm_workspace(M, N, 32))
                ws = _workspace(ws_n, x2.device) if ws_n else None
                nat.check(lib.hhb_gemm_f32a(M, N, k, x2.data_ptr(), k, wa.data_ptr(), wa[:, 2 * kp:].data_ptr(),
                                            wa.stride(0), b32.data_ptr(), y.data_ptr(), N, 0, D.ptr(ws), None, 0, 0,
                                            _stream()), "DenseLayer")
            else:
                xa, _ = split3_padded(x2, 0)
                y = gemm(xa, wa, 3 * kp, bias=b32)
            y = y.reshape(*xd.shape[:-1], y.shape[-1])
        else:
            # float64 (the reference's own precision, learn.py:210-211): a plain
            # library DGEMM -- no tensor-core form keeps 53 mantissa bits
            w = _dev(self.weights).to(xd.dtype)
            b = _dev(self.bias).to(xd.dtype)
            y = torch.matmul(xd, w.t()) + b
        return y if on_dev else y.cpu().numpy()

    @staticmethod
    def init(n_out: int, n_in: int, rng: np.random.Generator, scale: float | None = None) -> "DenseLayer":
        s = 1.0 / math.sqrt(n_in) if scale is None else scale
        return DenseLayer(rng.normal(0.0, s, size=(n_out, n_in)), np.zeros(n_out))


def _readout_ws(n_in: int, dev) -> torch.Tensor:
    nbytes = int(nat.load().hhb_readout_workspace(nat.F64, n_in))
    key = (dev, nbytes)
    ws = _READOUT_WS.get(key)
    if ws is None:
        ws = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
        _READOUT_WS[key] = ws
    return ws


_READOUT_WS: dict = {}


def _x3(filtered) -> torch.Tensor:
    """(B, T, C) float64 device tensor with unit channel stride (views kept)."""
    x = _dev(filtered).double()
    if x.dim() != 3:
        raise UsageError("filtered inputs must be (batch, steps, channels)")
    return x if x.stride(2) == 1 else x.contiguous()


def _readout_drive(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """dense(filtered)[..., 0] written time-major (T, B): the HH i_series."""
    B, T, C = x.shape
    out = torch.empty((T, B), dtype=torch.float64, device=x.device)
    nat.check(nat.load().hhb_readout_drive(nat.F64, B, T, C, x.data_ptr(), x.stride(0), x.stride(1),
                                           w.data_ptr(), b.data_ptr(), out.data_ptr(), D.stream()),
              "hhb_readout_drive")
    return out


@dataclass
class ReadoutModel:
    """PSP filter -> dense dendrite layer -> HH point neuron -> affine output
    scaling (learn.py:223-274).  The dendrite GEMV and its weight gradient are
    hhb_readout_drive / hhb_readout_grad, the neuron is the fused forward and
    BPTT kernels; numpy in -> numpy out like the reference, CUDA tensors in ->
    tensors out (what `fit` uses so the whole loop stays on the device)."""

    dense: DenseLayer
    scale_w: float
    scale_b: float
    neuron: object
    kernel: PSPKernel

    def filter_inputs(self, spikes):
        """spikes (B, T, C) -> filtered currents (B, T, C) (learn.py:233-235)."""
        on_dev = D.is_dev(spikes)
        x = _dev(spikes).double().permute(1, 0, 2).contiguous()     # (T, B, C)
        y = psp_filter(x, self.kernel).permute(1, 0, 2)              # (B, T, C) view
        return y if on_dev else y.cpu().numpy()

    def _params_dev(self, dev):
        w = _dev(self.dense.weights).double().reshape(-1).contiguous()
        b = _dev(self.dense.bias).double().reshape(-1).contiguous()
        if b.numel() != 1:
            raise UsageError("ReadoutModel has one output channel")
        return w, b

    def _drive(self, filtered):
        x = _x3(filtered)
        w, b = self._params_dev(x.device)
        if w.numel() != x.shape[2]:
            raise UsageError("dense weights do not match the channel count")
        return x, _readout_drive(x, w, b)

    def forward(self, filtered):
        """filtered (B, T, C) -> (prediction (B, T), membrane (B, T)) (learn.py:237-245)."""
        from .dynamics import init_state, simulate
        on_dev = D.is_dev(filtered)
        _, i_series = self._drive(filtered)                         # (T, B)
        state0 = init_state(self.neuron, i_series.shape[1:], device=i_series.device)
        trace = simulate(self.neuron, i_series, state0=state0)
        v = trace.v_series.double().t()                              # (B, T)
        pred = v * _scalar(self.scale_w, v) + _scalar(self.scale_b, v)
        if on_dev:
            return pred, v
        return pred.cpu().numpy(), v.contiguous().cpu().numpy()

    def params(self) -> dict:
        return {"w": self.dense.weights, "b": self.dense.bias,
                "scale_w": self.scale_w if D.is_dev(self.scale_w) else np.float64(self.scale_w),
                "scale_b": self.scale_b if D.is_dev(self.scale_b) else np.float64(self.scale_b)}

    def load_params(self, p: dict) -> None:
        """learn.py:255-259; device tensors are kept on the device."""
        if D.is_dev(p["w"]):
            self.dense.weights, self.dense.bias = p["w"], p["b"]
            self.scale_w, self.scale_b = p["scale_w"], p["scale_b"]
            return
        self.dense.weights = np.asarray(p["w"], dtype=np.float64)
        self.dense.bias = np.asarray(p["b"], dtype=np.float64)
        self.scale_w = float(p["scale_w"])
        self.scale_b = float(p["scale_b"])

    def grads(self, filtered, seed_pred, v, surrogate=None) -> dict:
        """d(loss)/d(prediction) -> every trainable (learn.py:261-274)."""
        from .adjoint import backward_through_time
        from .dynamics import init_state
        on_dev = D.is_dev(filtered)
        sp = _dev(seed_pred).double()
        vd = _dev(v).double()
        d_scale_w = (sp * vd).sum()
        d_scale_b = sp.sum()
        seed_v = (sp * _scalar(self.scale_w, sp)).t().contiguous()  # (T, B)
        x, i_series = self._drive(filtered)
        state0 = init_state(self.neuron, i_series.shape[1:], device=i_series.device)
        res = backward_through_time(self.neuron, state0, i_series, seed_v, surrogate=surrogate)
        d_i = res.d_i.double().contiguous()                          # (T, B) = d_drive time-major
        B, T, C = x.shape
        d_w = torch.empty((1, C), dtype=torch.float64, device=x.device)
        d_b = torch.empty(1, dtype=torch.float64, device=x.device)
        ws = _readout_ws(C, x.device)
        nat.check(nat.load().hhb_readout_grad(nat.F64, B, T, C, x.data_ptr(), x.stride(0), x.stride(1),
                                              d_i.data_ptr(), d_w.data_ptr(), d_b.data_ptr(), ws.data_ptr(),
                                              ws.numel() * 8, D.stream()), "hhb_readout_grad")
        if on_dev:
            return {"w": d_w, "b": d_b, "scale_w": d_scale_w, "scale_b": d_scale_b}
        return {"w": d_w.cpu().numpy(), "b": d_b.cpu().numpy(), "scale_w": float(d_scale_w.item()),
                "scale_b": float(d_scale_b.item())}


def _scalar(s, like: torch.Tensor):
    return s.to(like.dtype) if isinstance(s, torch.Tensor) else float(s)


@dataclass
class TeacherStudentTask:
    """Frozen teacher readout labelling Poisson spike trains (learn.py:277-286)."""

    teacher: ReadoutModel
    train_inputs: np.ndarray   # (B, T, C) binary
    train_targets: np.ndarray  # (B, T)
    val_inputs: np.ndarray
    val_targets: np.ndarray
    pad_len: int


def make_teacher_student_task(n_channels: int = 64, n_steps: int = 500, n_train: int = 16, n_val: int = 8,
                              rate_hz: float = 60.0, pad_len: int = 50, seed: int = 0,
                              neuron=None) -> TeacherStudentTask:
    """The synthetic fitting task (learn.py:289-327): signed teacher weights
    (first half excitatory U(0.5, 1.5), second half inhibitory -U(0.1, 0.6),
    scaled by 16 / n_channels, bias 0.45) and Bernoulli(rate·dt) spike trains,
    drawn from default_rng(seed) in the reference's order; targets from the
    teacher's device forward."""
    from .defaults import cortical_rs_params
    rng = np.random.default_rng(seed)
    neuron = cortical_rs_params(dt=0.1) if neuron is None else neuron
    kernel = PSPKernel(tau_decay=2.0, length=64, dt=neuron.dt)
    n_exc = n_channels // 2
    w = np.empty((1, n_channels))
    w[0, :n_exc] = rng.uniform(0.5, 1.5, n_exc)
    w[0, n_exc:] = -rng.uniform(0.1, 0.6, n_channels - n_exc)
    w *= 16.0 / n_channels
    teacher = ReadoutModel(DenseLayer(w, np.array([0.45])), 1.0, 0.0, neuron, kernel)
    p_spike = rate_hz * neuron.dt / 1000.0
    train_inputs = (rng.random((n_train, n_steps, n_channels)) < p_spike).astype(np.float64)
    val_inputs = (rng.random((n_val, n_steps, n_channels)) < p_spike).astype(np.float64)
    train_targets, _ = teacher.forward(teacher.filter_inputs(train_inputs))
    val_targets, _ = teacher.forward(teacher.filter_inputs(val_inputs))
    return TeacherStudentTask(teacher, train_inputs, train_targets, val_inputs, val_targets, pad_len)


def make_student(task: TeacherStudentTask, seed: int = 1) -> ReadoutModel:
    """Teacher architecture with re-initialised trainables (learn.py:330-336)."""
    rng = np.random.default_rng(seed)
    t = task.teacher
    n_in = np.shape(t.dense.weights)[1]
    return ReadoutModel(DenseLayer.init(1, n_in, rng, scale=4.0 / n_in), 1.0, 0.0, t.neuron, t.kernel)


@dataclass
class TrainConfig:
    epochs: int = 200
    lr: float = 5e-4
    cosine: bool = True
    freeze: bool = False


def evaluate_smape(model: ReadoutModel, inputs, targets, pad_len: int) -> float:
    """sMAPE of the model's prediction past the warm-up prefix (learn.py:346-348)."""
    pred, _ = model.forward(model.filter_inputs(inputs))
    return smape(_dev(pred)[:, pad_len:], _dev(targets)[:, pad_len:])


def fit(model: ReadoutModel, task: TeacherStudentTask, config: TrainConfig):
    """Full-batch fitting loop (learn.py:351-377), device-resident.  Returns
    the history rows (epoch, train_loss, val_smape); the model ends with numpy
    parameters as the reference's.

    Same arithmetic as the reference's loop, fewer passes: the training and
    validation samples are filtered once and simulated as ONE population per
    epoch (the validation forward of epoch e uses the parameters loaded at the
    start of epoch e, exactly as the training forward does, and the neurons are
    independent), and that forward also writes the per-step checkpoints the
    BPTT kernel reads instead of re-simulating (backward_through_time with
    plan=None recomputes the same states).  Parameters and Adam moments stay
    on the device; each epoch reads back one small vector (loss, validation
    sMAPE, overflow flags), and the errors are raised in the reference's
    order: NumericalOverflowError (training forward), TrainingDivergedError,
    GradientOverflowError, NumericalOverflowError (validation forward)."""
    from .adjoint import _backward, default_surrogate
    from .dynamics import _forward, init_state
    from .errors import GradientOverflowError, NumericalOverflowError
    dev = D.require_cuda()
    xt = np.asarray(task.train_inputs, dtype=np.float64)
    xv = np.asarray(task.val_inputs, dtype=np.float64)
    B, Bv = xt.shape[0], xv.shape[0]
    n_all = B + Bv
    x_all = _x3(model.filter_inputs(torch.as_tensor(np.concatenate([xt, xv], 0), device=dev)))
    T = x_all.shape[1]
    targets = _dev(task.train_targets).double()
    val_targets = _dev(task.val_targets).double()
    pad = task.pad_len
    mask = torch.zeros_like(targets)
    mask[:, pad:] = 1.0
    masked_targets = targets * mask
    neuron = model.neuron
    ng = neuron.n_gates
    s0 = init_state(neuron, (n_all,), device=dev)
    v0, g0 = s0.v.reshape(n_all), s0.gates.reshape(ng, n_all)
    v_out = torch.empty((T, n_all), dtype=v0.dtype, device=dev)
    ckpt = torch.empty((T, 1 + ng, n_all), dtype=v0.dtype, device=dev)
    adj_v = torch.empty(B, dtype=v0.dtype, device=dev)
    adj_g = torch.empty((ng, B), dtype=v0.dtype, device=dev)
    d_w = torch.empty((1, x_all.shape[2]), dtype=torch.float64, device=dev)
    d_b = torch.empty(1, dtype=torch.float64, device=dev)
    ws = _readout_ws(x_all.shape[2], dev)
    sur = default_surrogate(neuron)
    opt = AdamState(lr=config.lr)
    params = {k: _dev(v).double() for k, v in model.params().items()}
    history = []

    def host_params(p):
        return {k: (t.cpu().numpy() if t.dim() else np.float64(t.item())) for k, t in p.items()}

    def first_bad_step(v_part):                                            # (T, n) -> first bad t
        ok = torch.isfinite(v_part).all(dim=1)
        return int(torch.nonzero(~ok)[0, 0].item()) if not bool(ok.all().item()) else None

    for epoch in range(config.epochs):
        model.load_params(params)
        w, b = model._params_dev(dev)
        cur = _readout_drive(x_all, w, b).to(v0.dtype)                      # (T, B + Bv)
        _, _, fbad = _forward(neuron, v0, g0, cur, n_all, 1, T, v_out=v_out, ckpt=ckpt, ckpt_every=1)
        v_all = v_out.double().t()                                          # (B + Bv, T)
        pred_all = v_all * params["scale_w"] + params["scale_b"]
        loss, seed = mse_loss(pred_all[:B] * mask, masked_targets)
        gbad = None
        if not config.freeze:
            seed_m = seed * mask
            v = v_all[:B]
            grads = {"scale_w": (seed_m * v).sum(), "scale_b": seed_m.sum()}
            seed_v = (seed_m * params["scale_w"]).t().contiguous().to(v0.dtype)   # (T, B)
            adj_v.zero_()
            adj_g.zero_()
            d_i, _, gbad = _backward(neuron, sur, cur, n_all, 1, T, B, ckpt, 1, seed_v, None, adj_v, adj_g,
                                     ck_ld=n_all)
            d_i = d_i.double()
            nat.check(nat.load().hhb_readout_grad(nat.F64, B, T, x_all.shape[2], x_all.data_ptr(), x_all.stride(0),
                                                  x_all.stride(1), d_i.data_ptr(), d_w.data_ptr(), d_b.data_ptr(),
                                                  ws.data_ptr(), ws.numel() * 8, D.stream()), "hhb_readout_grad")
            grads["w"], grads["b"] = d_w, d_b
            lr = cosine_lr(config.lr, epoch, config.epochs) if config.cosine else config.lr
            new_params = adam_step(params, grads, opt, lr=lr)
        val = _smape_dev(pred_all[B:, pad:], val_targets[:, pad:])
        flags = torch.cat([t.double().reshape(1) for t in
                           (loss, val, fbad != D.INT64_MAX, gbad if gbad is not None else torch.full_like(fbad, -1))])
        loss_f, val_f, fb, gb = flags.cpu().tolist()
        if fb:
            step = first_bad_step(v_out[:, :B])
            if step is not None:
                model.load_params(host_params(params))
                raise NumericalOverflowError("membrane potential became non-finite", step)
        if not math.isfinite(loss_f):
            model.load_params(host_params(params))
            raise TrainingDivergedError("training loss became non-finite", epoch)
        if gb >= 0:
            model.load_params(host_params(params))
            raise GradientOverflowError("adjoint state became non-finite", int(gb))
        if fb:
            model.load_params(host_params(params))
            raise NumericalOverflowError("membrane potential became non-finite", first_bad_step(v_out[:, B:]))
        if not config.freeze:
            params = new_params
        history.append((epoch, loss_f, val_f))
    model.load_params(host_params(params))
    return history


# ---------------------------------------------------------------------------
# dataset and history files (learn.py:384-414)
# ---------------------------------------------------------------------------


def write_ndjson_dataset(path, inputs, targets, pad_len: int) -> None:
    """One JSON record per sample: {"input": 2-D, "target": 2-D, "pad_len"} (learn.py:384-395)."""
    with open(path, "w") as f:
        for x, y in zip(inputs, targets):
            y = np.asarray(y)
            tgt = y.reshape(-1, 1) if y.ndim == 1 else y
            f.write(json.dumps({"input": np.asarray(x).tolist(), "target": tgt.tolist(),
                                "pad_len": pad_len}) + "\n")


def read_ndjson_dataset(path):
    """(inputs, targets, pad_len) stacked from write_ndjson_dataset's format (learn.py:398-408)."""
    xs, ys, pad = [], [], 0
    with open(path) as f:
        for line in f:
            if line.strip():
                rec = json.loads(line)
                xs.append(np.asarray(rec["input"], dtype=np.float64))
                ys.append(np.asarray(rec["target"], dtype=np.float64))
                pad = int(rec["pad_len"])
    return np.stack(xs), np.stack(ys), pad


def write_history_csv(path, history) -> None:
    """epoch,train_loss,val_smape with repr floats (learn.py:411-415)."""
    with open(path, "w") as f:
        f.write("epoch,train_loss,val_smape\n")
        for epoch, loss, val in history:
            f.write(f"{epoch},{loss!r},{val!r}\n")
