"""Drop-in for `hhengine.dynamics`: channel definitions, neuron state, the fused
HH step and the step loop -- executed by the sm_100a kernels of libhhb200.so.

Same names, signatures, argument meaning and exceptions as the reference
module (hhengine/dynamics.py).  What changes is where the work runs:

  * `simulate` (dynamics.py:541-586) is ONE `hhb_forward` launch: all T steps
    are fused in registers, V is written once per step, spikes as a bitmap.
  * `hh_step` (dynamics.py:443-529) is the same launch with T = 1.
  * the elementary ops (gate_rates, gate_step, ionic_current, spike_detect)
    and RateFn evaluation are small device kernels built on the same math.

Array convention: numpy in -> numpy out (host<->device copies inside the
call, reference semantics); CUDA tensors in -> CUDA tensors out (the
device-resident path a PyTorch user or the training layer uses).
Arithmetic: HHParams.dtype float64 (the reference default) selects the parity
build, which follows the reference's operation order; float32 selects the
throughput build (MUFU exp/rcp; tolerance documented in DESIGN.md).
"""

from __future__ import annotations

import ctypes as C
import functools
import math
from dataclasses import dataclass, replace
from typing import Sequence

import numpy as np
import torch

from . import _device as D
from . import _native as nat
from .errors import ConfigurationError, NumericalOverflowError, UsageError

# Below this |denominator| the linoid rate switches to its analytic limit
# (dynamics.py:24-25); honoured bit-for-bit by the float64 build.
LINOID_EPS = 1e-7


# ---------------------------------------------------------------------------
# channel description (dynamics.py:32-224)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class RateFn:
    """alpha(V) or beta(V): "linoid" a*x/(1-exp(-x/b)), "exp" a*exp(-x/b),
    "sigmoid" a/(1+exp(-x/b)), with x = V - v0 (dynamics.py:32-54)."""

    kind: str
    a: float
    v0: float
    b: float

    def __post_init__(self):
        if self.kind not in nat.RATE_KIND:
            raise ConfigurationError(f"unknown rate kind {self.kind!r}")
        if self.b == 0.0:
            raise ConfigurationError("rate slope parameter b must be nonzero")

    def _eval(self, v, slope: int):
        out_np = not D.is_dev(v)
        dtype = np.float64 if out_np else D.np_dtype(v.dtype)
        vd = D.to_dev(v, dtype)
        out = torch.empty_like(vd)
        r = nat.pack_rate(self)
        nat.check(nat.load().hhb_rate_eval(C.byref(r), slope, D.code(dtype), vd.numel(),
                                           vd.data_ptr(), out.data_ptr(), D.stream()),
                  "rate evaluation")
        return _back(out, out_np, np.ndim(v) == 0 if out_np else False)

    def __call__(self, v):
        return self._eval(v, 0)

    def deriv(self, v):
        """d(rate)/dV, analytic (dynamics.py:67-79)."""
        return self._eval(v, 1)

    def to_dict(self) -> dict:
        return {"kind": self.kind, "a": self.a, "v0": self.v0, "b": self.b}

    @staticmethod
    def from_dict(d: dict) -> "RateFn":
        try:
            return RateFn(str(d["kind"]), float(d["a"]), float(d["v0"]), float(d["b"]))
        except KeyError as k:
            raise ConfigurationError(f"rate function missing key {k}") from None


@dataclass(frozen=True)
class GateSpec:
    """Gating sub-unit with rates alpha/beta and its integer power in the
    channel conductance (dynamics.py:96-125)."""

    name: str
    alpha: RateFn
    beta: RateFn
    exponent: int = 1

    def __post_init__(self):
        if self.exponent < 0 or int(self.exponent) != self.exponent:
            raise ConfigurationError(f"gate {self.name}: exponent must be a non-negative integer")

    def to_dict(self) -> dict:
        return {"name": self.name, "exponent": self.exponent,
                "alpha": self.alpha.to_dict(), "beta": self.beta.to_dict()}

    @staticmethod
    def from_dict(d: dict) -> "GateSpec":
        return GateSpec(name=str(d["name"]), alpha=RateFn.from_dict(d["alpha"]),
                        beta=RateFn.from_dict(d["beta"]), exponent=int(d.get("exponent", 1)))


@dataclass(frozen=True)
class ChannelSpec:
    """g_max * prod p_i^k_i * (V - e_rev); empty gates = leak (dynamics.py:128-159)."""

    name: str
    g_max: float
    e_rev: float
    gates: tuple = ()

    def __post_init__(self):
        if self.g_max < 0:
            raise ConfigurationError(f"channel {self.name}: g_max must be >= 0")

    def to_dict(self) -> dict:
        return {"name": self.name, "g_max": self.g_max, "e_rev": self.e_rev,
                "gates": [g.to_dict() for g in self.gates]}

    @staticmethod
    def from_dict(d: dict) -> "ChannelSpec":
        return ChannelSpec(name=str(d["name"]), g_max=float(d["g_max"]), e_rev=float(d["e_rev"]),
                           gates=tuple(GateSpec.from_dict(g) for g in d.get("gates", [])))


@dataclass(frozen=True)
class HHParams:
    """Conductance-based point neuron (dynamics.py:162-224).  rate_scale
    multiplies every alpha and beta.  dtype picks the device arithmetic."""

    c_m: float
    channels: tuple
    v_rest: float
    v_theta: float
    dt: float
    rate_scale: float = 1.0
    dtype: type = np.float64

    def __post_init__(self):
        if self.c_m <= 0:
            raise ConfigurationError("c_m must be > 0")
        if self.dt <= 0:
            raise ConfigurationError("dt must be > 0")
        if self.rate_scale <= 0:
            raise ConfigurationError("rate_scale must be > 0")
        names = [c.name for c in self.channels]
        if len(set(names)) != len(names):
            raise ConfigurationError(f"channel names must be unique, got {names}")
        object.__setattr__(self, "channels", tuple(self.channels))

    @property
    def gate_layout(self) -> tuple:
        """(channel_index, gate) pairs in declaration order = gate-row order."""
        return tuple((ci, g) for ci, ch in enumerate(self.channels) for g in ch.gates)

    @property
    def n_gates(self) -> int:
        return sum(len(ch.gates) for ch in self.channels)

    def with_(self, **kw) -> "HHParams":
        return replace(self, **kw)

    def to_dict(self) -> dict:
        return {"c_m": self.c_m, "dt": self.dt, "v_rest": self.v_rest, "v_theta": self.v_theta,
                "rate_scale": self.rate_scale, "channels": [c.to_dict() for c in self.channels]}

    @staticmethod
    def from_dict(d: dict) -> "HHParams":
        try:
            return HHParams(c_m=float(d["c_m"]),
                            channels=tuple(ChannelSpec.from_dict(c) for c in d["channels"]),
                            v_rest=float(d.get("v_rest", -65.0)),
                            v_theta=float(d.get("v_theta", 0.0)), dt=float(d["dt"]),
                            rate_scale=float(d.get("rate_scale", 1.0)))
        except KeyError as k:
            raise ConfigurationError(f"neuron parameters missing key {k}") from None


@dataclass(frozen=True)
class LIFParams:
    """Dimensionless LIF baseline (dynamics.py:227-244)."""

    tau: float
    v_theta: float
    v_reset: float
    dt: float
    dtype: type = np.float64

    def __post_init__(self):
        if self.tau <= 0:
            raise ConfigurationError("tau must be > 0")
        if self.v_theta <= self.v_reset:
            raise ConfigurationError("v_theta must exceed v_reset")
        if self.dt <= 0:
            raise ConfigurationError("dt must be > 0")


@functools.lru_cache(maxsize=256)
def _table(params: HHParams) -> nat.Params:
    return nat.pack_hh(params)


# ---------------------------------------------------------------------------
# state containers (dynamics.py:250-299)
# ---------------------------------------------------------------------------

@dataclass
class NeuronState:
    """v: batch shape S; gates: (n_gates,) + S in gate_layout order."""

    v: object
    gates: object

    def copy(self) -> "NeuronState":
        return NeuronState(_copy(self.v), _copy(self.gates))


@dataclass
class Trace:
    """Time-major record: v_series and spike_series are (T,) + S."""

    v_series: object
    spike_series: object
    dt: float

    def __post_init__(self):
        if tuple(self.v_series.shape) != tuple(self.spike_series.shape):
            raise UsageError("v_series and spike_series must share shape")

    @property
    def n_steps(self) -> int:
        return int(self.v_series.shape[0])

    def spike_count(self):
        return self.spike_series.sum(axis=0)

    def spike_times(self, dt_offset: float = 1.0) -> np.ndarray:
        """Spike times (ms) of a single-neuron trace: (index + dt_offset) * dt."""
        if self.v_series.ndim != 1:
            raise UsageError("spike_times requires a single-neuron trace")
        return (np.flatnonzero(_np(self.spike_series)) + dt_offset) * self.dt

    def to_csv(self, path) -> None:
        """Columns t_ms, neuron_id, v_mV, spike; one row per neuron per step."""
        v = _np(self.v_series).reshape(self.n_steps, -1).astype(np.float64, copy=False)
        s = _np(self.spike_series).reshape(self.n_steps, -1)
        with open(path, "w") as f:
            f.write("t_ms,neuron_id,v_mV,spike\n")
            for t in range(self.n_steps):
                t_ms = (t + 1) * self.dt
                for n in range(v.shape[1]):
                    f.write(f"{t_ms:.6g},{n},{v[t, n]!r},{int(s[t, n])}\n")


def _np(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _copy(x):
    return x.clone() if isinstance(x, torch.Tensor) else np.array(x, copy=True)


def _back(t: torch.Tensor, to_numpy: bool, scalar: bool = False, dtype=None):
    if not to_numpy:
        return t
    a = D.to_host(t, dtype)
    return a[()] if scalar else a


def init_state(params, shape: tuple = (), v0: float | None = None, device=None) -> NeuronState:
    """Rest state: V = v0 (default v_rest), every gate at alpha/(alpha+beta)
    of that potential, 0.5 where the total rate is 0 (dynamics.py:302-317).

    The steady-state rates are evaluated by the device rate kernel in float64.
    device=None returns numpy arrays (reference behaviour); a torch device
    returns CUDA tensors.
    """
    shape = tuple(shape)
    if isinstance(params, LIFParams):
        if device is None:
            v = np.full(shape, 0.0 if v0 is None else v0, dtype=params.dtype)
            return NeuronState(v, np.zeros((0,) + shape, dtype=params.dtype))
        td = D.torch_dtype(params.dtype)
        return NeuronState(torch.full(shape, 0.0 if v0 is None else float(v0), dtype=td, device=device),
                           torch.zeros((0,) + shape, dtype=td, device=device))
    if v0 is None:
        v0 = params.v_rest
    fracs = steady_state_gates(params, v0)
    if device is None:
        v = np.full(shape, v0, dtype=params.dtype)
        gates = np.empty((len(fracs),) + shape, dtype=params.dtype)
        for gi, f in enumerate(fracs):
            gates[gi] = f
        return NeuronState(v, gates)
    td = D.torch_dtype(params.dtype)
    v = torch.full(shape, float(v0), dtype=td, device=device)
    gates = torch.empty((len(fracs),) + shape, dtype=td, device=device)
    for gi, f in enumerate(fracs):
        gates[gi].fill_(f)
    return NeuronState(v, gates)


def steady_state_gates(params: HHParams, v0: float) -> list:
    """Per-gate open fraction alpha/(alpha+beta) at v0 (0.5 for zero rate);
    memoised per (channel table, v0): every init_state of a population
    otherwise pays one rate launch and read-back per gate."""
    try:
        key = (params, float(v0))
        hit = _STEADY.get(key)
    except TypeError:
        key, hit = None, None
    if hit is None:
        hit = _steady_state_gates(params, v0)
        if key is not None:
            if len(_STEADY) > 256:
                _STEADY.clear()
            _STEADY[key] = hit
    return list(hit)


_STEADY: dict = {}


def _steady_state_gates(params: HHParams, v0: float) -> tuple:
    out = []
    for _, gate in params.gate_layout:
        a, b = gate_rates(gate, np.float64(v0), params.rate_scale)
        a, b = float(a), float(b)
        s = a + b
        out.append(a / s if s > 0 else 0.5)
    return tuple(out)


# ---------------------------------------------------------------------------
# elementary operations (dynamics.py:324-381), device kernels
# ---------------------------------------------------------------------------

def gate_rates(gate: GateSpec, v, rate_scale: float = 1.0):
    """(alpha(V), beta(V)) times rate_scale, finite at removable singularities."""
    out_np = not D.is_dev(v)
    dtype = np.float64 if out_np else D.np_dtype(v.dtype)
    vd = D.to_dev(v, dtype)
    a, b = torch.empty_like(vd), torch.empty_like(vd)
    g = nat.pack_gate(gate)
    nat.check(nat.load().hhb_gate_rates(C.byref(g), float(rate_scale), D.code(dtype), vd.numel(),
                                        vd.data_ptr(), a.data_ptr(), b.data_ptr(), D.stream()),
              "gate_rates")
    scalar = out_np and np.ndim(v) == 0
    return _back(a, out_np, scalar), _back(b, out_np, scalar)


def gate_step(p, alpha, beta, dt: float):
    """Exponential Euler p_inf + (p - p_inf) exp(-dt (alpha+beta)); p_inf = p
    where the total rate is not positive (dynamics.py:335-346)."""
    out_np = not any(D.is_dev(x) for x in (p, alpha, beta))
    dtype = np.float64 if out_np else D.np_dtype(next(x.dtype for x in (p, alpha, beta) if D.is_dev(x)))
    shape = np.broadcast_shapes(np.shape(p), np.shape(alpha), np.shape(beta))
    pd, ad, bd = (D.to_dev(x, dtype).expand(shape).contiguous() for x in (p, alpha, beta))
    out = torch.empty(shape, dtype=pd.dtype, device=pd.device)
    nat.check(nat.load().hhb_gate_step(D.code(dtype), out.numel(), pd.data_ptr(), ad.data_ptr(),
                                       bd.data_ptr(), float(dt), out.data_ptr(), D.stream()),
              "gate_step")
    return _back(out, out_np, out_np and len(shape) == 0)


def int_pow(p, k: int):
    """p**k by left-fold multiplication (dynamics.py:349-357)."""
    if k == 0:
        return torch.ones_like(p) if isinstance(p, torch.Tensor) else np.ones_like(p)
    out = p
    for _ in range(k - 1):
        out = out * p
    return out


def ionic_current(state: NeuronState, channels: Sequence[ChannelSpec]):
    """sum_X g_X prod p^k (V - E_X) over `channels` (dynamics.py:360-376)."""
    n_gates = sum(len(ch.gates) for ch in channels)
    if int(state.gates.shape[0]) != n_gates:
        raise ConfigurationError(
            f"state carries {state.gates.shape[0]} gates but channels define {n_gates}")
    P = nat.pack_params(tuple(channels))
    out_np = not D.is_dev(state.v)
    dtype = np.float64 if out_np else D.np_dtype(state.v.dtype)
    vd = D.to_dev(state.v, dtype).reshape(-1)
    n = vd.numel()
    gd = D.to_dev(state.gates, dtype).reshape(n_gates, n) if n_gates else None
    out = torch.empty_like(vd)
    nat.check(nat.load().hhb_ionic_current(C.byref(P), D.code(dtype), n, vd.data_ptr(),
                                           D.ptr(gd), n, out.data_ptr(), D.stream()),
              "ionic_current")
    shape = tuple(np.shape(state.v)) if out_np else tuple(state.v.shape)
    return _back(out.reshape(shape), out_np, out_np and len(shape) == 0)


def spike_detect(v_prev, v_new, v_theta: float):
    """Upward threshold crossing v_prev < v_theta <= v_new (dynamics.py:379-381)."""
    out_np = not (D.is_dev(v_prev) or D.is_dev(v_new))
    dtype = np.float64 if out_np else D.np_dtype((v_prev if D.is_dev(v_prev) else v_new).dtype)
    shape = np.broadcast_shapes(np.shape(v_prev), np.shape(v_new))
    a, b = (D.to_dev(x, dtype).expand(shape).contiguous() for x in (v_prev, v_new))
    out = torch.empty(shape, dtype=torch.uint8, device=a.device)
    nat.check(nat.load().hhb_spike_detect(D.code(dtype), out.numel(), a.data_ptr(), b.data_ptr(),
                                          float(v_theta), out.data_ptr(), D.stream()),
              "spike_detect")
    res = out.view(torch.bool)
    if not out_np:
        return res
    r = D.to_host(res)
    return r[()] if len(shape) == 0 else r


# ---------------------------------------------------------------------------
# fused HH step and step loop
# ---------------------------------------------------------------------------

class Workspace:
    """Caller-owned device scratch reused across hh_step calls (the role of
    the reference Workspace, dynamics.py:388-406): the first-bad-step word,
    the spike bitmap row and the unpacked spike bytes of one step."""

    def __init__(self, shape: tuple, dtype=np.float64):
        n = int(np.prod(shape, dtype=np.int64))
        self.size = n
        self.dtype = dtype
        dev = D.require_cuda()
        self.first_bad = torch.empty(1, dtype=torch.int64, device=dev)
        self.bits = torch.empty(max(1, (n + 31) // 32), dtype=torch.int32, device=dev)
        self.spikes = torch.empty(max(1, n), dtype=torch.uint8, device=dev)

    def matches(self, shape, dtype) -> bool:
        return self.size == int(np.prod(shape, dtype=np.int64)) and np.dtype(self.dtype) == np.dtype(dtype)


def _forward(params: HHParams, v: torch.Tensor, g: torch.Tensor, cur: torch.Tensor, i_st: int,
             i_sn: int, steps: int, *, v_fin=None, g_fin=None, v_out=None, bits=None,
             ckpt=None, ckpt_every: int = 0, step_base: int = 0, first_bad=None,
             reset_bad: bool = True, spk_val=None, step_dev=None, sq_part=None, spk_bf16=None):
    """One hhb_forward launch on device tensors (flat v (n,), g (ng, n)).
    first_bad accumulates (atomicMin) across launches when reset_bad=False.
    spk_bf16: optional (steps, n) bf16 tensor receiving the spike flags as 0/1."""
    n = v.numel()
    P = _table(params)
    dt = D.code(v.dtype)
    v_fin = v_fin if v_fin is not None else torch.empty_like(v)
    g_fin = g_fin if g_fin is not None else torch.empty_like(g)
    if first_bad is None:
        first_bad = torch.empty(1, dtype=torch.int64, device=v.device)
        reset_bad = True
    if reset_bad:
        first_bad.fill_(D.INT64_MAX)
    words = (n + 31) // 32
    rc = nat.load().hhb_forward_ex2(
        C.byref(P), dt, n, steps, v.data_ptr(), D.ptr(g) if g.numel() else None, n,
        v_fin.data_ptr(), D.ptr(g_fin) if g_fin.numel() else None,
        D.ptr(cur), i_st, i_sn,
        D.ptr(v_out), n, D.ptr(bits), words, D.ptr(spk_val), n,
        D.ptr(ckpt), max(1, ckpt_every), n,
        step_base, first_bad.data_ptr(), D.ptr(step_dev), D.ptr(sq_part), D.ptr(spk_bf16), n, D.stream())
    nat.check(rc, "hhb_forward")
    return v_fin, g_fin, first_bad


def _raise_if_bad(first_bad: torch.Tensor, step_index=None, offset: int = 0):
    bad = int(first_bad.item())
    if bad != D.INT64_MAX:
        raise NumericalOverflowError("membrane potential became non-finite",
                                     bad - offset if step_index is None else step_index)


def _unpack(bits: torch.Tensor, steps: int, n: int, out: torch.Tensor | None = None) -> torch.Tensor:
    words = (n + 31) // 32
    if out is None:
        out = torch.empty((steps, n), dtype=torch.uint8, device=bits.device)
    nat.check(nat.load().hhb_unpack_spikes(bits.data_ptr(), words, steps, n, out.data_ptr(), n,
                                           D.stream()), "unpack spikes")
    return out.view(torch.bool)


def hh_step(state: NeuronState, i_ext, params: HHParams, workspace: Workspace | None = None,
            step_index: int | None = None, out_state: NeuronState | None = None):
    """One fused forward step (dynamics.py:443-529): gates and I_ion read the
    pre-update V and gates; returns (new state, spikes).  Raises
    NumericalOverflowError(step_index) on a non-finite V'."""
    if isinstance(params, LIFParams):
        return lif_step(state, i_ext, params)
    on_dev = D.is_dev(state.v)
    shape = tuple(state.v.shape) if on_dev else np.shape(state.v)
    dtype = D.np_dtype(state.v.dtype) if on_dev else np.asarray(state.v).dtype
    if dtype not in (np.float32, np.float64):
        dtype = np.dtype(np.float64)
    n = int(np.prod(shape, dtype=np.int64))
    ng = int(state.gates.shape[0])
    if ng != params.n_gates:
        raise ConfigurationError(f"state carries {ng} gates but channels define {params.n_gates}")
    ws = workspace if (workspace is not None and workspace.matches(shape, dtype)) else Workspace(shape, dtype)
    v = D.to_dev(state.v, dtype).reshape(-1)
    g = D.to_dev(state.gates, dtype).reshape(ng, n)
    i_arr = i_ext if D.is_dev(i_ext) else np.asarray(i_ext, dtype=dtype)
    i_shape = tuple(i_arr.shape)
    if i_shape == tuple(shape):
        cur, i_sn = D.to_dev(i_arr, dtype).reshape(-1), 1
    elif len(i_shape) == 0 or int(np.prod(i_shape)) == 1:
        cur, i_sn = D.to_dev(i_arr, dtype).reshape(1), 0
    else:
        cur, i_sn = D.to_dev(i_arr, dtype).expand(shape).contiguous().reshape(-1), 1
    dev_out = on_dev and out_state is not None and D.is_dev(out_state.v)
    v_fin = out_state.v.reshape(-1) if dev_out and out_state.v.is_contiguous() else None
    g_fin = out_state.gates.reshape(ng, n) if dev_out and out_state.gates.is_contiguous() else None
    v_fin, g_fin, bad = _forward(params, v, g, cur, 0, i_sn, 1, v_fin=v_fin, g_fin=g_fin,
                                 bits=ws.bits, step_base=0 if step_index is None else step_index,
                                 first_bad=ws.first_bad)
    _raise_if_bad(bad, step_index)
    spikes = _unpack(ws.bits.view(1, -1), 1, n, ws.spikes[:n].view(1, n)).reshape(shape)
    if on_dev:
        new = NeuronState(v_fin.reshape(shape), g_fin.reshape((ng,) + tuple(shape)))
        if out_state is not None and not dev_out:
            out_state.v[...] = D.to_host(new.v)
            out_state.gates[...] = D.to_host(new.gates)
            return out_state, spikes.clone()
        if out_state is not None:
            if out_state.v.data_ptr() != v_fin.data_ptr():
                out_state.v.copy_(new.v)
            if out_state.gates.data_ptr() != g_fin.data_ptr():
                out_state.gates.copy_(new.gates)
            return out_state, spikes.clone()
        return new, spikes.clone()
    v_np = D.to_host(v_fin).reshape(shape)
    g_np = D.to_host(g_fin).reshape((ng,) + tuple(shape))
    sp = D.to_host(spikes).reshape(shape)
    if out_state is None:
        return NeuronState(v_np, g_np), (sp[()] if len(shape) == 0 else sp)
    out_state.v[...] = v_np
    out_state.gates[...] = g_np
    return out_state, (sp[()] if len(shape) == 0 else sp)


def _lif_run(params: LIFParams, v: torch.Tensor, cur: torch.Tensor, steps: int, i_st: int, i_sn: int,
             record: bool):
    """hhb_lif_forward on device tensors: v (n,), cur flat; returns (v_fin, V, spikes)."""
    n = v.numel()
    v_fin = torch.empty_like(v)
    vs = torch.empty((steps, n), dtype=v.dtype, device=v.device) if record else None
    ss = torch.empty((steps, n), dtype=torch.uint8, device=v.device)
    nat.check(nat.load().hhb_lif_forward(D.code(v.dtype), n, steps, params.tau, params.dt, params.v_theta,
                                         params.v_reset, v.data_ptr(), cur.data_ptr(), i_st, i_sn, D.ptr(vs),
                                         ss.data_ptr(), v_fin.data_ptr(), D.stream()), "hhb_lif_forward")
    return v_fin, vs, ss.view(torch.bool)


def lif_step(state: NeuronState, i, params: LIFParams):
    """Leaky integration with inclusive threshold and hard reset (dynamics.py:532-538)."""
    on_dev = D.is_dev(state.v)
    dev = D.require_cuda()
    # numpy inputs compute in NumPy's promoted type, as the reference does
    # (a float64 current promotes a float32 LIF state)
    dt_ = params.dtype if on_dev else np.result_type(np.asarray(state.v).dtype, np.asarray(i).dtype)
    v = D.to_dev(state.v, dt_, dev)
    shape = tuple(v.shape)
    cur = D.to_dev(i, dt_, dev)
    i_sn = 0 if cur.numel() == 1 else 1
    if i_sn:
        cur = cur.expand(shape).contiguous()
    v_fin, _, ss = _lif_run(params, v.reshape(-1).contiguous(), cur.reshape(-1), 1, 0, i_sn, False)
    v_out, spikes = v_fin.reshape(shape), ss[0].reshape(shape)
    if on_dev:
        return NeuronState(v_out, state.gates), spikes
    return NeuronState(D.to_host(v_out), state.gates), D.to_host(spikes)


def simulate(params, i_series, state0: NeuronState | None = None, record_state: bool = False):
    """Run T steps over the time-major current series (dynamics.py:541-586) in
    ONE fused kernel launch.  Deterministic: identical arguments give
    bit-identical traces.  Returns the Trace (and the final state when
    record_state is set).  numpy input -> numpy Trace with float64 v_series
    (as the reference); CUDA tensor input -> CUDA tensors in params.dtype."""
    if isinstance(params, LIFParams):
        return _simulate_lif(params, i_series, state0, record_state)
    on_dev = D.is_dev(i_series)
    dtype = np.dtype(params.dtype)
    shape_all = tuple(i_series.shape) if on_dev else np.shape(i_series)
    T = int(shape_all[0]) if len(shape_all) else 0
    shape = tuple(shape_all[1:])
    n = int(np.prod(shape, dtype=np.int64))
    ng = params.n_gates
    if state0 is None:
        # built on the device even for numpy calls: only the final state, if
        # requested, travels back to the host
        state0 = init_state(params, shape, device=D.require_cuda() if (on_dev or T > 0) else None)
    elif tuple(state0.v.shape) != shape and T > 0:
        raise UsageError(f"state shape {tuple(state0.v.shape)} does not match input shape {shape}")
    else:
        # the reference's hh_step computes in the state's dtype (dynamics.py:459,
        # :564-566): a float32 state0 runs float32 arithmetic even with float64
        # params, and vice versa
        sd = _state_dtype(state0.v)
        if sd is not None and sd != dtype:
            params = params.with_(dtype=sd)
            dtype = sd
    if T == 0:
        empty_v = (torch.empty((0,) + shape, dtype=D.torch_dtype(dtype), device=D.require_cuda())
                   if on_dev else np.empty((0,) + shape, dtype=np.float64))
        empty_s = (torch.empty((0,) + shape, dtype=torch.bool, device=empty_v.device)
                   if on_dev else np.empty((0,) + shape, dtype=bool))
        tr = Trace(empty_v, empty_s, params.dt)
        return (tr, state0) if record_state else tr
    dev = D.require_cuda()
    v = D.to_dev(state0.v, dtype, dev).reshape(n)
    g = D.to_dev(state0.gates, dtype, dev).reshape(ng, n)
    if not on_dev and T * n >= _PIPELINE_MIN_ELEMS:
        return _simulate_pipelined(params, np.asarray(i_series).reshape(T, n), v, g, T, shape, record_state)
    cur = D.to_dev(i_series, dtype, dev).reshape(T, n)
    v_out = torch.empty((T, n), dtype=cur.dtype, device=dev)
    bits = torch.empty((T, (n + 31) // 32), dtype=torch.int32, device=dev)
    v_fin, g_fin, bad = _forward(params, v, g, cur, n, 1, T, v_out=v_out, bits=bits)
    _raise_if_bad(bad)
    spikes = _unpack(bits, T, n)
    if on_dev:
        tr = Trace(v_out.reshape((T,) + shape), spikes.reshape((T,) + shape), params.dt)
        fin = NeuronState(v_fin.reshape(shape), g_fin.reshape((ng,) + shape))
    else:
        tr = Trace(D.to_host(v_out, np.float64).reshape((T,) + shape),
                   D.to_host(spikes).reshape((T,) + shape), params.dt)
        fin = NeuronState(D.to_host(v_fin).reshape(shape), D.to_host(g_fin).reshape((ng,) + shape))
    if record_state:
        return tr, fin
    return tr


_PIPELINE_MIN_ELEMS = 1 << 22


def _state_dtype(v):
    """float32 / float64 of a state array or tensor, None for anything else."""
    try:
        d = D.np_dtype(v.dtype) if isinstance(v, torch.Tensor) else np.dtype(np.asarray(v).dtype)
    except Exception:
        return None
    return d if d in (np.dtype(np.float32), np.dtype(np.float64)) else None


def _simulate_pipelined(params, i2, v, g, T, shape, record_state):
    """numpy-in/numpy-out simulate for large calls: time chunks with host
    copy, H2D, kernel and D2H overlapped (see _pipeline.py)."""
    from . import _pipeline
    n = v.numel()
    ng = g.shape[0]
    first_bad = torch.full((1,), D.INT64_MAX, dtype=torch.int64, device=v.device)

    def fwd(cur, tc, v_out, bits, t0):
        _forward(params, v, g, cur, n, 1, tc, v_fin=v, g_fin=g, v_out=v_out, bits=bits, step_base=t0,
                 first_bad=first_bad, reset_bad=False)

    def unpack(bits, tc, nn, out):
        _unpack(bits, tc, nn, out)

    vs, ss = _pipeline.simulate_host(params, i2, v, g, fwd, unpack)
    _raise_if_bad(first_bad)
    tr = Trace(vs.reshape((T,) + shape), ss.reshape((T,) + shape), params.dt)
    if record_state:
        return tr, NeuronState(D.to_host(v).reshape(shape), D.to_host(g).reshape((ng,) + shape))
    return tr


def _simulate_lif(params: LIFParams, i_series, state0, record_state):
    """All T LIF steps in one hhb_lif_forward launch."""
    on_dev = D.is_dev(i_series)
    shape_all = tuple(i_series.shape) if on_dev else np.shape(i_series)
    T, shape = int(shape_all[0]), tuple(shape_all[1:])
    dev = D.require_cuda()
    # the reference casts the series to float64 (dynamics.py:552), so its LIF
    # arithmetic is float64 whatever params.dtype says; device tensors keep
    # params.dtype
    cdt = params.dtype if on_dev else np.float64
    cur = D.to_dev(i_series, cdt, dev)
    n = int(np.prod(shape, dtype=np.int64)) if shape else 1
    state = state0 if state0 is not None else init_state(params, shape, device=dev)
    v0 = D.to_dev(state.v, cdt, dev).reshape(n).contiguous()
    cur = cur.reshape(T, n).contiguous()
    v_fin, vs, ss = _lif_run(params, v0, cur, T, n, 1, True)
    vs, ss = vs.reshape((T,) + shape), ss.reshape((T,) + shape)
    st = NeuronState(v_fin.reshape(shape), state.gates)
    if on_dev:
        tr = Trace(vs, ss, params.dt)
    else:
        tr = Trace(D.to_host(vs, np.float64), D.to_host(ss), params.dt)
        st = NeuronState(D.to_host(st.v), state.gates)
    return (tr, st) if record_state else tr


def firing_rate(trace: Trace):
    """Mean rate in Hz per batch element (dynamics.py:589-594)."""
    if trace.n_steps == 0:
        return np.zeros(tuple(trace.v_series.shape[1:]))
    duration_ms = trace.n_steps * trace.dt
    return trace.spike_count() * 1000.0 / duration_ms


def isi_cv(trace: Trace) -> float:
    """ISI coefficient of variation of a single-neuron trace (dynamics.py:597-603)."""
    times = trace.spike_times()
    if times.size < 3:
        return float("nan")
    isi = np.diff(times)
    return float(np.std(isi) / np.mean(isi))
