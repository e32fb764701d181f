"""Drop-in for `hhengine.adjoint`: surrogate gradients, the exact adjoint of the
fused HH step, checkpoint plans and BPTT -- executed by libhhb200.so.

`backward_through_time` (adjoint.py:281-365) is two launches:
  1. hhb_forward with checkpoints every K steps (K = plan.segment_length, or 1
     for the plan-less full-storage mode: every state is kept, as the
     reference's `stored` dict does),
  2. hhb_backward, which walks the segments newest first, recomputes each
     segment's states from its checkpoint (bit-identical to step 1: same
     device function, explicit rounding) and applies the exact adjoint step
     (adjoint.py:116-188) per neuron in registers.  Parameter gradients are
     reduced per block and summed in a fixed order (deterministic).
Gradients do not depend on the plan -- in this implementation bit-for-bit.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as nat
from .dynamics import HHParams, LIFParams, NeuronState, _forward, _raise_if_bad, _table
from .errors import GradientOverflowError, UsageError


# ---------------------------------------------------------------------------
# surrogate (adjoint.py:33-66)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SurrogateSpec:
    """Smooth stand-in for the spike indicator's derivative: kinds
    "sigmoid-derivative" (default) and "rectangular" (adjoint.py:33-48)."""

    kind: str = "sigmoid-derivative"
    width: float = 1.0

    def __post_init__(self):
        if self.kind not in nat.SUR_KIND:
            raise UsageError(f"unknown surrogate kind {self.kind!r}")
        if self.width <= 0:
            raise UsageError("surrogate width must be > 0")


def default_surrogate(params) -> SurrogateSpec:
    """Width = a quarter of the neuron's threshold scale (adjoint.py:51-57)."""
    if isinstance(params, HHParams):
        scale = abs(params.v_theta - params.v_rest)
    else:
        scale = abs(params.v_theta - params.v_reset)
    return SurrogateSpec("sigmoid-derivative", 0.25 * max(scale, 1e-12))


def surrogate_grad(u, spec: SurrogateSpec):
    """Surrogate kernel at threshold offsets u = V' - v_theta (adjoint.py:60-66)."""
    out_np = not D.is_dev(u)
    dtype = np.float64 if out_np else D.np_dtype(u.dtype)
    ud = D.to_dev(u, dtype)
    out = torch.empty_like(ud)
    s = nat.pack_surrogate(spec)
    nat.check(nat.load().hhb_surrogate_grad(C.byref(s), D.code(dtype), ud.numel(), ud.data_ptr(),
                                            out.data_ptr(), D.stream()), "surrogate_grad")
    if not out_np:
        return out
    a = D.to_host(out)
    return a[()] if np.ndim(u) == 0 else a


# ---------------------------------------------------------------------------
# adjoint state (adjoint.py:73-99)
# ---------------------------------------------------------------------------

@dataclass
class AdjointState:
    """dL/dV, dL/dgates per neuron plus the c_m / g_max accumulators."""

    d_v: object
    d_gates: object
    d_c_m: float = 0.0
    d_g_max: object = None
    d_spike: object = None

    @staticmethod
    def zeros(state: NeuronState, n_channels: int) -> "AdjointState":
        if D.is_dev(state.v):
            return AdjointState(torch.zeros_like(state.v), torch.zeros_like(state.gates), 0.0,
                                np.zeros(n_channels))
        return AdjointState(np.zeros_like(state.v), np.zeros_like(state.gates), 0.0, np.zeros(n_channels))

    def copy(self) -> "AdjointState":
        def cp(x):
            if x is None:
                return None
            return x.clone() if isinstance(x, torch.Tensor) else np.array(x, copy=True)
        return AdjointState(cp(self.d_v), cp(self.d_gates), self.d_c_m, cp(self.d_g_max), cp(self.d_spike))


# ---------------------------------------------------------------------------
# device driver shared by hh_step_backward and backward_through_time
# ---------------------------------------------------------------------------

def _backward(params, spec, cur, i_st, i_sn, T, n, ckpt, K, seed_v, seed_s, adj_v, adj_g,
              d_i=None, step_base=0, want_d_i=True, split=None, d_sum=None, ck_ld=None, sv_ld=None,
              sv_scale=None):
    """One hhb_backward(_ex) launch; returns (d_i or None, d_params np.array[1+nch], first_bad).

    split = (hi, lo[, group, pitch]) bf16 [T][ld] tensors receive dI as bf16 hi/lo halves
    (neuron i at (i // group) * pitch + i % group when group > 0)
    and d_sum [n] float accumulates the per-neuron sums of dI (SNN layer).
    ck_ld: leading dimension of the checkpoint planes (default n) -- the first
    n neurons of a wider forward's checkpoints.  sv_ld: seed_v row stride
    (default n); sv_scale: device float multiplying seed_v as it is read."""
    dev = adj_v.device
    ng = params.n_gates
    nch = len(params.channels)
    P = _table(params)
    S = nat.pack_surrogate(spec)
    dt = D.code(adj_v.dtype)
    lib = nat.load()
    seg = torch.empty((K, 1 + ng, n), dtype=adj_v.dtype, device=dev) if K > 1 else None
    parts = torch.empty(int(lib.hhb_backward_partials(n, dt)), dtype=torch.float64, device=dev)
    d_params = torch.zeros(1 + nch, dtype=torch.float64, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    if d_i is None and want_d_i:
        d_i = torch.empty((T, n), dtype=adj_v.dtype, device=dev)
    hi, lo = (split[0], split[1]) if split is not None else (None, None)
    grp, pitch = (split[2], split[3]) if split is not None and len(split) > 2 else (0, 0)
    ld_split = hi.shape[-1] if hi is not None else n
    rc = lib.hhb_backward_ex(
        C.byref(P), C.byref(S), dt, n, T, cur.data_ptr(), i_st, i_sn,
        ckpt.data_ptr(), K, n if ck_ld is None else ck_ld, D.ptr(seg),
        D.ptr(seed_v), n if sv_ld is None else sv_ld, D.ptr(seed_s), n,
        adj_v.data_ptr(), D.ptr(adj_g) if ng else None, n,
        D.ptr(d_i), n, d_params.data_ptr(), parts.data_ptr(),
        step_base, bad.data_ptr(), D.ptr(hi), D.ptr(lo), ld_split, grp, pitch, D.ptr(d_sum), D.ptr(sv_scale),
        D.stream())
    nat.check(rc, "hhb_backward")
    return d_i, d_params, bad


def _raise_if_grad_bad(bad: torch.Tensor, step_index=None):
    b = int(bad.item())
    if b >= 0:
        raise GradientOverflowError("adjoint state became non-finite",
                                    b if step_index is None else step_index)


def hh_step_backward(state_in: NeuronState, i_ext, params: HHParams, adj_out: AdjointState,
                     surrogate: SurrogateSpec, step_index: int | None = None):
    """Adjoint of one fused step (adjoint.py:102-194).  state_in is the step's
    exact input; adj_out carries dL/dV', dL/dp' and optionally dL/dspike.
    Returns (adj_in, d_i_ext)."""
    if isinstance(params, LIFParams):
        return lif_step_backward(state_in, i_ext, params, adj_out, surrogate, step_index)
    on_dev = D.is_dev(state_in.v)
    shape = tuple(state_in.v.shape) if on_dev else np.shape(state_in.v)
    n = int(np.prod(shape, dtype=np.int64))
    ng = params.n_gates
    dtype = np.dtype(params.dtype) if not on_dev else D.np_dtype(state_in.v.dtype)
    dev = D.require_cuda()
    ckpt = torch.empty((1, 1 + ng, n), dtype=D.torch_dtype(dtype), device=dev)
    ckpt[0, 0] = D.to_dev(state_in.v, dtype, dev).reshape(n)
    if ng:
        ckpt[0, 1:] = D.to_dev(state_in.gates, dtype, dev).reshape(ng, n)
    i_arr = i_ext if D.is_dev(i_ext) else np.asarray(i_ext, dtype=np.float64)
    if tuple(i_arr.shape) == tuple(shape):
        cur, i_sn = D.to_dev(i_arr, dtype, dev).reshape(n), 1
    elif int(np.prod(tuple(i_arr.shape))) == 1:
        cur, i_sn = D.to_dev(i_arr, dtype, dev).reshape(1), 0
    else:
        cur, i_sn = D.to_dev(i_arr, dtype, dev).expand(shape).contiguous().reshape(n), 1
    adj_v = D.to_dev(adj_out.d_v, dtype, dev).reshape(n).clone()
    adj_g = D.to_dev(adj_out.d_gates, dtype, dev).reshape(ng, n).clone()
    seed_s = None
    if adj_out.d_spike is not None:
        seed_s = D.to_dev(adj_out.d_spike, dtype, dev).expand(shape).contiguous().reshape(1, n)
    d_i, d_params, bad = _backward(params, surrogate, cur, 0, i_sn, 1, n, ckpt, 1, None, seed_s,
                                   adj_v, adj_g, step_base=0 if step_index is None else step_index)
    _raise_if_grad_bad(bad, step_index)
    dp = D.to_host(d_params)
    base_g = np.zeros(len(params.channels)) if adj_out.d_g_max is None else np.asarray(adj_out.d_g_max, dtype=np.float64)
    d_c_m = float(adj_out.d_c_m) + float(dp[0])
    d_g_max = base_g + dp[1:]
    if on_dev:
        adj_in = AdjointState(adj_v.reshape(shape), adj_g.reshape((ng,) + tuple(shape)), d_c_m, d_g_max)
        return adj_in, d_i.reshape(shape)
    adj_in = AdjointState(D.to_host(adj_v, np.float64).reshape(shape),
                          D.to_host(adj_g, np.float64).reshape((ng,) + tuple(shape)), d_c_m, d_g_max)
    return adj_in, D.to_host(d_i, np.float64).reshape(shape)


def lif_step_backward(state_in: NeuronState, i_ext, params: LIFParams, adj_out: AdjointState,
                      surrogate: SurrogateSpec, step_index: int | None = None):
    """Adjoint of one LIF step with the surrogate reset factor (adjoint.py:197-227),
    float64 as in the reference, one hhb_lif_backward launch."""
    on_dev = D.is_dev(state_in.v)
    dev = D.require_cuda()
    v = D.to_dev(state_in.v, np.float64, dev)
    shape = tuple(v.shape)
    n = v.numel()
    cur = D.to_dev(i_ext, np.float64, dev)
    i_sn = 0 if cur.numel() == 1 else 1
    if i_sn:
        cur = cur.expand(shape).contiguous()
    g_out = D.to_dev(adj_out.d_v, np.float64, dev).expand(shape).contiguous()
    g_sp = (D.to_dev(adj_out.d_spike, np.float64, dev).expand(shape).contiguous()
            if adj_out.d_spike is not None else None)
    d_v_in = torch.empty(shape, dtype=torch.float64, device=dev)
    d_i = torch.empty(shape, dtype=torch.float64, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    S = nat.pack_surrogate(surrogate)
    nat.check(nat.load().hhb_lif_backward(D.code(torch.float64), n, params.tau, params.dt, params.v_theta,
                                          params.v_reset, C.byref(S), v.contiguous().data_ptr(), cur.data_ptr(),
                                          i_sn, g_out.data_ptr(), D.ptr(g_sp), d_v_in.data_ptr(), d_i.data_ptr(),
                                          bad.data_ptr(), D.stream()), "hhb_lif_backward")
    if int(bad.item()) >= 0:
        raise GradientOverflowError("adjoint state became non-finite", step_index)
    zeros_g = torch.zeros_like(D.to_dev(adj_out.d_gates, np.float64, dev))
    if on_dev:
        return AdjointState(d_v_in, zeros_g, adj_out.d_c_m, adj_out.d_g_max), d_i
    return (AdjointState(D.to_host(d_v_in), D.to_host(zeros_g), adj_out.d_c_m, adj_out.d_g_max),
            D.to_host(d_i))


# ---------------------------------------------------------------------------
# checkpoint plans (adjoint.py:234-278)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class CheckpointPlan:
    """Forward state indices retained for the backward pass (adjoint.py:234-247)."""

    total_steps: int
    segment_length: int
    stored_indices: tuple

    def __post_init__(self):
        if not self.stored_indices or self.stored_indices[0] != 0:
            raise UsageError("stored_indices must cover step 0")
        gaps = np.diff(np.asarray(tuple(self.stored_indices) + (self.total_steps,)))
        if gaps.size and gaps.max() > self.segment_length:
            raise UsageError("checkpoint gap exceeds segment_length")


def make_plan(total_steps: int, budget: int) -> CheckpointPlan:
    """Equal spacing, segment_length = ceil(T / budget) (adjoint.py:250-258)."""
    if total_steps < 1:
        raise UsageError("total_steps must be >= 1")
    if budget < 1:
        raise UsageError("budget must be >= 1")
    seg = math.ceil(total_steps / budget)
    return CheckpointPlan(total_steps, seg, tuple(range(0, total_steps, seg)))


@dataclass
class BPTTStats:
    """Forward-step count and peak retained states (adjoint.py:261-270)."""

    forward_calls: int = 0
    peak_stored_states: int = 0

    def observe(self, live: int):
        self.peak_stored_states = max(self.peak_stored_states, live)


@dataclass
class BPTTResult:
    d_i: object
    d_state0: AdjointState
    d_c_m: float
    d_g_max: object
    stats: BPTTStats


def _plan_stats(T: int, K: int, full: bool) -> BPTTStats:
    """What the two launches did, in the reference's counting
    (adjoint.py:310-348): forward steps executed and the peak number of
    NeuronStates resident (checkpoints + one recomputed segment)."""
    st = BPTTStats()
    if full:
        st.forward_calls = T
        st.observe(T + 1)
        return st
    lows = list(range(0, T, K))
    st.forward_calls = T
    st.observe(len(lows))
    live = len(lows)
    for lo in reversed(lows):
        hi = min(lo + K, T)
        st.forward_calls += hi - lo - 1
        st.observe(live + (hi - lo) - 1)
        live -= 1
    return st


def backward_through_time(params: HHParams, state0: NeuronState, i_series, seed_v,
                          seed_spike=None, plan: CheckpointPlan | None = None,
                          surrogate: SurrogateSpec | None = None) -> BPTTResult:
    """Reverse-mode sweep over the simulated chain (adjoint.py:281-365).

    seed_v[t] is dL/dV of trace row t, seed_spike[t] dL/dspike.  Gradients do
    not depend on the plan; the plan bounds the resident states (here: the
    checkpoint buffer [ceil(T/K), 1+n_gates, n] plus one segment buffer).
    """
    on_dev = D.is_dev(i_series)
    shape_all = tuple(i_series.shape) if on_dev else np.shape(i_series)
    T = int(shape_all[0])
    shape = tuple(shape_all[1:])
    n = int(np.prod(shape, dtype=np.int64))
    sv_shape = tuple(seed_v.shape) if D.is_dev(seed_v) else np.shape(seed_v)
    if sv_shape[0] != T:
        raise UsageError(f"seed series length {sv_shape[0]} != input length {T}")
    if seed_spike is not None:
        ss_shape = tuple(seed_spike.shape) if D.is_dev(seed_spike) else np.shape(seed_spike)
        if ss_shape[0] != T:
            raise UsageError("seed_spike length mismatch")
    if surrogate is None:
        surrogate = default_surrogate(params)
    if plan is not None and plan.total_steps != T:
        raise UsageError("plan total_steps does not match input length")
    ng = params.n_gates
    nch = len(params.channels)
    full = plan is None
    K = 1 if full else max(1, min(int(plan.segment_length), T))
    stats = _plan_stats(T, K, full)
    dtype = np.dtype(params.dtype) if not on_dev else D.np_dtype(i_series.dtype)
    dev = D.require_cuda()
    if T == 0:
        zero = AdjointState.zeros(state0, nch)
        return BPTTResult(np.empty((0,) + shape), zero, 0.0, np.zeros(nch), stats)

    cur = D.to_dev(i_series, dtype, dev).reshape(T, n)
    v0 = D.to_dev(state0.v, dtype, dev).reshape(n)
    g0 = D.to_dev(state0.gates, dtype, dev).reshape(ng, n)
    nck = (T + K - 1) // K
    ckpt = torch.empty((nck, 1 + ng, n), dtype=cur.dtype, device=dev)
    _, _, bad = _forward(params, v0, g0, cur, n, 1, T, ckpt=ckpt, ckpt_every=K)
    _raise_if_bad(bad)

    sv = D.to_dev(seed_v, dtype, dev).reshape(T, n)
    ss = None if seed_spike is None else D.to_dev(seed_spike, dtype, dev).reshape(T, n)
    adj_v = torch.zeros(n, dtype=cur.dtype, device=dev)
    adj_g = torch.zeros((ng, n), dtype=cur.dtype, device=dev)
    d_i, d_params, gbad = _backward(params, surrogate, cur, n, 1, T, n, ckpt, K, sv, ss, adj_v, adj_g)
    _raise_if_grad_bad(gbad)
    dp = D.to_host(d_params)
    d_c_m, d_g_max = float(dp[0]), dp[1:].copy()
    if on_dev:
        d0 = AdjointState(adj_v.reshape(shape), adj_g.reshape((ng,) + shape), d_c_m, d_g_max)
        return BPTTResult(d_i.reshape((T,) + shape), d0, d_c_m, d_g_max, stats)
    d0 = AdjointState(D.to_host(adj_v, np.float64).reshape(shape),
                      D.to_host(adj_g, np.float64).reshape((ng,) + shape), d_c_m, d_g_max)
    return BPTTResult(D.to_host(d_i, np.float64).reshape((T,) + shape), d0, d_c_m, d_g_max, stats)
