"""CPU oracle for the HH hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain NumPy, the algorithm of the reference package
`hhengine` (arXiv 2601.21407, BrainFuse desk-scale re-implementation) for the
hot path named in BASELINE.json `north_star`:

  * rate functions and their analytic slopes   (dynamics.py:56-79)
  * steady-state initial gates                 (dynamics.py:302-317)
  * the fused forward step                     (dynamics.py:443-529, _rate_into :409-440)
  * the step loop                              (dynamics.py:541-586)
  * surrogate gradient                         (adjoint.py:51-66)
  * the adjoint step                           (adjoint.py:102-194)
  * checkpoint plans + BPTT driver             (adjoint.py:250-258, :281-365)
  * ring-buffer spike delivery                 (cortex.py:239-310)
  * dense projection + readout gradient        (learn.py:210-211, :264-274)

Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` may import this module, and only as the checker
or the timed CPU baseline -- never as the product.  The product path
(`paper_2601_21407_b200`) runs on the GPU through the C-ABI library and raises
if that library is missing.

Parity pinning: every function here is checked against golden vectors produced
by running the reference itself in the build container (oracle/make_golden.py
-> tests/golden/*.npz, see tests/test_oracle_golden.py).

Parameter objects are duck-typed: anything with the attribute layout of the
reference `HHParams` (c_m, dt, v_rest, v_theta, rate_scale, channels[].g_max,
.e_rev, .gates[].alpha/.beta(.kind,.a,.v0,.b), .exponent) works -- both the
reference's own dataclasses and the product's mirrors.
"""

from __future__ import annotations

import math

import numpy as np

SINGULAR_DEN = 1e-7  # dynamics.py:25 LINOID_EPS


# ---------------------------------------------------------------------------
# rates (dynamics.py:56-79 and the in-place order of _rate_into :409-440)
# ---------------------------------------------------------------------------

def rate_value(fn, v):
    """alpha/beta(V) for one RateFn; same op order as dynamics.py:56-65."""
    x = np.asarray(v, dtype=np.float64) - fn.v0
    arg = -x / fn.b
    if fn.kind == "exp":
        return fn.a * np.exp(arg)
    if fn.kind == "sigmoid":
        return fn.a / (1.0 + np.exp(arg))
    den = 1.0 - np.exp(arg)
    with np.errstate(divide="ignore", invalid="ignore"):
        val = fn.a * x / den
    return np.where(np.abs(den) < SINGULAR_DEN, fn.a * fn.b, val)


def rate_slope(fn, v):
    """d rate / dV, dynamics.py:67-79."""
    x = np.asarray(v, dtype=np.float64) - fn.v0
    ex = np.exp(-x / fn.b)
    if fn.kind == "exp":
        return -(fn.a / fn.b) * ex
    if fn.kind == "sigmoid":
        sg = 1.0 / (1.0 + ex)
        return (fn.a / fn.b) * sg * (1.0 - sg)
    den = 1.0 - ex
    with np.errstate(divide="ignore", invalid="ignore"):
        val = fn.a * (den - x * ex / fn.b) / (den * den)
    return np.where(np.abs(den) < SINGULAR_DEN, 0.5 * fn.a, val)


def _rate_inplace(fn, v, out, tmp):
    """Restates _rate_into (dynamics.py:409-440) without the scale step; runs
    in the dtype of `out`, so the reference's float32 mode is reproducible."""
    np.subtract(v, fn.v0, out=tmp)
    np.negative(tmp, out=out)
    np.divide(out, fn.b, out=out)
    np.exp(out, out=out)
    if fn.kind == "exp":
        np.multiply(out, fn.a, out=out)
    elif fn.kind == "sigmoid":
        np.add(out, 1.0, out=out)
        np.divide(fn.a, out, out=out)
    else:
        np.subtract(1.0, out, out=out)
        singular = np.abs(out) < SINGULAR_DEN
        np.multiply(tmp, fn.a, out=tmp)
        with np.errstate(divide="ignore", invalid="ignore"):
            np.divide(tmp, out, out=out)
        if singular.any():
            np.copyto(out, fn.a * fn.b, where=singular)
    return out


def gate_list(params):
    """Flattened (channel_index, gate) order = gate-row order (dynamics.py:190-193)."""
    return [(ci, g) for ci, ch in enumerate(params.channels) for g in ch.gates]


# ---------------------------------------------------------------------------
# state init (dynamics.py:302-317)
# ---------------------------------------------------------------------------

def steady_gates(params, v0=None):
    """Per-gate scalar open fraction at v0 (fp64), 0.5 for zero total rate."""
    v0 = params.v_rest if v0 is None else v0
    vals = []
    for _, g in gate_list(params):
        a = rate_value(g.alpha, np.float64(v0))
        b = rate_value(g.beta, np.float64(v0))
        if params.rate_scale != 1.0:
            a, b = a * params.rate_scale, b * params.rate_scale
        s = a + b
        vals.append(float(a / s) if s > 0 else 0.5)
    return np.asarray(vals, dtype=np.float64)


def rest_state(params, n, v0=None, dtype=np.float64):
    v0 = params.v_rest if v0 is None else v0
    v = np.full((n,), v0, dtype=dtype)
    gates = np.empty((len(gate_list(params)), n), dtype=dtype)
    gates[:] = steady_gates(params, v0)[:, None]
    return v, gates


# ---------------------------------------------------------------------------
# fused forward step (dynamics.py:443-529)
# ---------------------------------------------------------------------------

class Overflow(Exception):
    def __init__(self, step):
        super().__init__(f"non-finite membrane potential at step {step}")
        self.step = step


class StepScratch:
    """Five flat scratch rows, the Workspace of dynamics.py:388-406."""

    def __init__(self, n, dtype=np.float64):
        self.n, self.dtype = n, np.dtype(dtype)
        self.r = np.empty((5, n), dtype=dtype)


def step(params, v, gates, i_ext, scratch=None, v_out=None, g_out=None, step_index=None):
    """One fused HH step on flat arrays; returns (v_new, gates_new, spikes).

    Arithmetic and its order follow hh_step (dynamics.py:472-528): gate update
    and ionic sum both use the pre-update V and gates; the total rate is
    guarded only at exactly zero (:494-508); the membrane update is
    V + (I - I_ion) * (dt / c_m) (:522-524).
    """
    n = v.shape[0]
    dtype = v.dtype
    if scratch is None or scratch.n != n or scratch.dtype != dtype:
        scratch = StepScratch(n, dtype)
    t0, t1, t2, eta, i_ion = scratch.r
    if v_out is None:
        v_out = np.empty_like(v)
    if g_out is None:
        g_out = np.empty_like(gates)
    dt, scale = params.dt, params.rate_scale
    i_ion.fill(0.0)
    row = 0
    for ch in params.channels:
        if not ch.gates:
            np.subtract(v, ch.e_rev, out=t0)
            np.multiply(t0, ch.g_max, out=t0)
            np.add(i_ion, t0, out=i_ion)
            continue
        eta.fill(1.0)
        for g in ch.gates:
            p = gates[row]
            if g.exponent == 1:
                np.multiply(eta, p, out=eta)
            elif g.exponent > 1:
                np.multiply(p, p, out=t2)
                for _ in range(g.exponent - 2):
                    np.multiply(t2, p, out=t2)
                np.multiply(eta, t2, out=eta)
            al = _rate_inplace(g.alpha, v, t0, t2)
            if scale != 1.0:
                np.multiply(al, scale, out=al)
            be = _rate_inplace(g.beta, v, t1, t2)
            if scale != 1.0:
                np.multiply(be, scale, out=be)
            np.add(al, be, out=be)                 # total rate s
            zero = None if be.all() else (be == 0.0)
            if zero is not None:
                np.copyto(be, 1.0, where=zero)
            np.divide(al, be, out=al)              # p_inf
            if zero is not None:
                np.copyto(be, 0.0, where=zero)
            np.multiply(be, -dt, out=be)
            np.exp(be, out=be)                     # decay
            dst = g_out[row]
            np.subtract(p, al, out=dst)
            np.multiply(dst, be, out=dst)
            np.add(dst, al, out=dst)
            if zero is not None:
                np.copyto(dst, p, where=zero)
            row += 1
        np.multiply(eta, ch.g_max, out=t1)
        np.subtract(v, ch.e_rev, out=t0)
        np.multiply(t1, t0, out=t0)
        np.add(i_ion, t0, out=i_ion)
    cur = np.asarray(i_ext, dtype=dtype)
    np.subtract(cur if cur.ndim == 0 else cur.reshape(-1), i_ion, out=t0)
    np.multiply(t0, params.dt / params.c_m, out=t0)
    np.add(v, t0, out=v_out)
    if not np.all(np.isfinite(v_out)):
        raise Overflow(step_index)
    spikes = (v < params.v_theta) & (v_out >= params.v_theta)
    return v_out, g_out, spikes


def simulate(params, i_series, v0=None, g0=None, dtype=np.float64, record_final=False):
    """Step loop of dynamics.py:541-586 (HH branch) on flat neuron arrays.

    i_series: (T, n). Returns (V (T, n) float64, spikes (T, n) bool[, v, g]).
    """
    i_series = np.asarray(i_series, dtype=np.float64)
    T, n = i_series.shape[0], int(np.prod(i_series.shape[1:], dtype=np.int64))
    i2 = i_series.reshape(T, n)
    if v0 is None:
        v, g = rest_state(params, n, dtype=dtype)
    else:
        v = np.asarray(v0, dtype=dtype).reshape(n).copy()
        g = np.asarray(g0, dtype=dtype).reshape(-1, n).copy()
    vs = np.empty((T, n), dtype=np.float64)
    ss = np.empty((T, n), dtype=bool)
    sc = StepScratch(n, dtype)
    bufs = [(np.empty_like(v), np.empty_like(g)), (np.empty_like(v), np.empty_like(g))]
    for t in range(T):
        vo, go = bufs[t % 2]
        v, g, sp = step(params, v, g, i2[t], sc, vo, go, step_index=t)
        vs[t] = v
        ss[t] = sp
    if record_final:
        return vs, ss, v.copy(), g.copy()
    return vs, ss


# ---------------------------------------------------------------------------
# surrogate (adjoint.py:51-66)
# ---------------------------------------------------------------------------

def default_width(params):
    return 0.25 * max(abs(params.v_theta - params.v_rest), 1e-12)


def surrogate(u, kind="sigmoid-derivative", width=1.0):
    u = np.asarray(u, dtype=np.float64)
    if kind == "rectangular":
        return np.where(np.abs(u) <= width, 0.5 / width, 0.0)
    s = 1.0 / (1.0 + np.exp(-u / width))
    return s * (1.0 - s) / width


# ---------------------------------------------------------------------------
# adjoint step (adjoint.py:102-194)
# ---------------------------------------------------------------------------

class GradOverflow(Exception):
    def __init__(self, step):
        super().__init__(f"non-finite adjoint at step {step}")
        self.step = step


def step_backward(params, v, gates, i_ext, d_v, d_gates, d_spike, sur_kind, sur_width,
                  step_index=None):
    """Adjoint of one step. Returns (d_v_in, d_gates_in, d_i, d_cm_inc, d_gmax_inc).

    Follows adjoint.py:116-194: recompute eta/drive/V' from the step input,
    fold the spike seed through the surrogate at V'-theta, then chain through
    the membrane update and the exponential-Euler gate update.
    """
    dt, cm, scale = params.dt, params.c_m, params.rate_scale
    dt_cm = dt / cm
    layout = gate_list(params)
    nch = len(params.channels)
    eta = np.empty((nch,) + v.shape)
    drive = np.empty((nch,) + v.shape)
    row = 0
    for ci, ch in enumerate(params.channels):
        e = 1.0
        for g in ch.gates:
            pk = gates[row] if g.exponent > 0 else np.ones_like(gates[row])
            for _ in range(g.exponent - 1):
                pk = pk * gates[row]
            e = e * pk
            row += 1
        eta[ci] = e
        drive[ci] = v - ch.e_rev
    gmax = np.array([ch.g_max for ch in params.channels])
    i_ion = np.einsum("c,c...->...", gmax, eta * drive)
    cur = np.asarray(i_ext, dtype=np.float64)
    v_new = v + dt_cm * (cur - i_ion)

    g_vp = d_v
    if d_spike is not None:
        g_vp = g_vp + d_spike * surrogate(v_new - params.v_theta, sur_kind, sur_width)

    d_i = g_vp * dt_cm
    d_cm_inc = float(np.sum(g_vp * (-(dt / cm ** 2)) * (cur - i_ion)))
    d_g_inc = np.array([float(np.sum(g_vp * (-dt_cm) * eta[c] * drive[c])) for c in range(nch)])

    d_v_in = g_vp * (1.0 - dt_cm * np.einsum("c,c...->...", gmax, eta))
    d_g_in = np.empty_like(d_gates, dtype=np.float64)
    row = 0
    for ci, ch in enumerate(params.channels):
        first = row
        for gj, g in enumerate(ch.gates):
            p = gates[row]
            a = rate_value(g.alpha, v) * scale
            b = rate_value(g.beta, v) * scale
            da = rate_slope(g.alpha, v) * scale
            db = rate_slope(g.beta, v) * scale
            s = a + b
            pos = s > 0
            s_safe = np.where(pos, s, 1.0)
            e = np.exp(-dt * s)
            pinf = np.where(pos, a / s_safe, p)
            up = d_gates[row]
            dp = up * np.where(pos, e, 1.0)
            dpinf = np.where(pos, (da * b - a * db) / (s_safe * s_safe), 0.0)
            dv_term = np.where(pos, dpinf * (1.0 - e) + (p - pinf) * (-dt * (da + db) * e), 0.0)
            d_v_in = d_v_in + up * dv_term
            k = g.exponent
            if k > 0:
                der = float(k) * (np.ones_like(p) if k == 1 else _ipow(p, k - 1))
                for oj, og in enumerate(ch.gates):
                    if oj != gj:
                        der = der * _ipow(gates[first + oj], og.exponent)
                dp = dp + g_vp * (-dt_cm) * ch.g_max * drive[ci] * der
            d_g_in[row] = dp
            row += 1
    if not (np.all(np.isfinite(d_v_in)) and np.all(np.isfinite(d_g_in))):
        raise GradOverflow(step_index)
    return d_v_in, d_g_in, d_i, d_cm_inc, d_g_inc


def _ipow(p, k):
    if k == 0:
        return np.ones_like(p)
    out = p
    for _ in range(k - 1):
        out = out * p
    return out


# ---------------------------------------------------------------------------
# plans + BPTT (adjoint.py:250-365)
# ---------------------------------------------------------------------------

def plan(total_steps, budget):
    """(segment_length, stored_indices) of adjoint.py:250-258."""
    if total_steps < 1 or budget < 1:
        raise ValueError("total_steps and budget must be >= 1")
    seg = math.ceil(total_steps / budget)
    return seg, tuple(range(0, total_steps, seg))


def bptt(params, v0, g0, i_series, seed_v, seed_spike=None, segment=None,
         sur_kind="sigmoid-derivative", sur_width=None):
    """Reverse sweep of adjoint.py:281-365 on flat arrays.

    segment=None is the full-storage mode; otherwise checkpoints every
    `segment` steps are recomputed per segment in reverse.  Returns a dict
    with d_i (T, n), d_v0, d_g0, d_c_m, d_g_max, forward_calls, peak_states.
    """
    if sur_width is None:
        sur_width = default_width(params)
    i_series = np.asarray(i_series, dtype=np.float64)
    T = i_series.shape[0]
    n = int(np.asarray(v0).size)
    i2 = i_series.reshape(T, n)
    sv = np.asarray(seed_v, dtype=np.float64).reshape(T, n)
    ssp = None if seed_spike is None else np.asarray(seed_spike, dtype=np.float64).reshape(T, n)
    calls = [0]

    def fwd(v, g, t):
        calls[0] += 1
        vn, gn, _ = step(params, v, g, i2[t], step_index=t)
        return vn, gn

    v = np.asarray(v0, dtype=np.float64).reshape(n)
    g = np.asarray(g0, dtype=np.float64).reshape(-1, n)
    if segment is None:
        states = [(v, g)]
        for t in range(T):
            states.append(fwd(*states[-1], t))
        peak = len(states)
        segs = [(0, T)]
        ckpt = None
    else:
        stored = set(range(0, T, segment))
        ckpt = {}
        cur = (v, g)
        for t in range(T):
            if t in stored:
                ckpt[t] = cur
            cur = fwd(*cur, t)
        peak = len(ckpt)
        bounds = sorted(ckpt) + [T]
        segs = [(bounds[k], bounds[k + 1]) for k in range(len(bounds) - 1)][::-1]
    d_v = np.zeros(n)
    d_g = np.zeros_like(g, dtype=np.float64)
    d_cm = 0.0
    d_gm = np.zeros(len(params.channels))
    d_i = np.empty((T, n))
    for lo, hi in segs:
        if ckpt is None:
            seg_states = states[lo:hi]
        else:
            seg_states = [ckpt[lo]]
            for t in range(lo, hi - 1):
                seg_states.append(fwd(*seg_states[-1], t))
            peak = max(peak, len(ckpt) + len(seg_states) - 1)
            ckpt.pop(lo)
        for t in range(hi - 1, lo - 1, -1):
            d_v = d_v + sv[t]
            sp = None if ssp is None else ssp[t]
            vs, gs = seg_states[t - lo]
            d_v, d_g, d_i[t], inc_cm, inc_g = step_backward(
                params, vs, gs, i2[t], d_v, d_g, sp, sur_kind, sur_width, step_index=t)
            d_cm += inc_cm
            d_gm = d_gm + inc_g
    return {"d_i": d_i, "d_v0": d_v, "d_g0": d_g, "d_c_m": d_cm, "d_g_max": d_gm,
            "forward_calls": calls[0], "peak_states": peak}


# ---------------------------------------------------------------------------
# dense projection + readout gradients (learn.py:210-211, :264-274)
# ---------------------------------------------------------------------------

def dense(x, w, b):
    return x @ w.T + b


def dense_grad_w(d_drive_btc, x_btk):
    """dW[c, k] = sum_{b,t} d_drive[b,t,c] x[b,t,k]; learn.py:272 generalised
    from one output channel to many."""
    return np.einsum("btc,btk->ck", d_drive_btc, x_btk)


def mse_loss(pred, target):
    """learn.py:80-88: mean squared error and its seed 2 (pred - target) / size."""
    diff = np.asarray(pred, np.float64) - np.asarray(target, np.float64)
    return float(np.mean(diff * diff)), 2.0 * diff / diff.size


def cross_entropy_loss(logits, target):
    """learn.py:92-107: softmax cross-entropy (mean over rows) and its seed."""
    z = np.asarray(logits, np.float64)
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    p = e / e.sum(axis=-1, keepdims=True)
    rows = np.arange(len(target))
    seed = p.copy()
    seed[rows, target] -= 1.0
    return float(-np.mean(np.log(p[rows, target]))), seed / len(target)


# ---------------------------------------------------------------------------
# network spike delivery (cortex.py:239-310)
# ---------------------------------------------------------------------------

class Ring:
    """SpikeBuffer of cortex.py:239-256."""

    def __init__(self, depth, n):
        self.depth = depth
        self.rows = np.zeros((depth, n))

    def push(self, t, targets, weights, delays):
        np.add.at(self.rows, ((t + delays) % self.depth, targets), weights)

    def pop(self, t):
        r = self.rows[t % self.depth]
        out = r.copy()
        r.fill(0.0)
        return out


def network_step(params, v, g, psp, ring, t, offsets, targets, weights, delays,
                 psp_decay, background=None, extra=None):
    """One step_network (cortex.py:273-310) with the background sample supplied
    by the caller instead of drawn from the RNG. Returns (v, g, psp, spikes)."""
    arrived = ring.pop(t)
    psp = psp * psp_decay
    psp = psp + arrived
    if background is not None:
        psp = psp + background
    cur = psp if extra is None else psp + extra
    v, g, spikes = step(params, v, g, cur, step_index=t)
    for s in np.flatnonzero(spikes):
        lo, hi = offsets[s], offsets[s + 1]
        if hi > lo:
            ring.push(t, targets[lo:hi], weights[lo:hi], delays[lo:hi])
    return v, g, psp, spikes


# ---------------------------------------------------------------------------
# multicompartment neurons (morphology.py:115-166)
# ---------------------------------------------------------------------------

def morph_axial(v, edges):
    """axial_current (morphology.py:115-124): v (n_comp, ...), edges
    [(i, j, g)] in declaration order; out[i] += g (v_j - v_i), out[j] -= it."""
    out = np.zeros_like(v)
    for i, j, g in edges:
        flow = g * (v[j] - v[i])
        out[i] += flow
        out[j] -= flow
    return out


def morph_simulate(params_list, edges, i_series, dtype=np.float64):
    """simulate_morphology (morphology.py:144-166) for compartments with
    channel tables params_list (graph order); i_series (T, n_comp) + batch.
    Returns (V (T, n_comp) + batch float64, spikes bool)."""
    i_series = np.asarray(i_series, dtype=np.float64)
    T, nc = i_series.shape[:2]
    shape = i_series.shape[2:]
    n = int(np.prod(shape, dtype=np.int64)) if shape else 1
    vs, gs = [], []
    for p in params_list:
        v, g = rest_state(p, n, dtype=dtype)
        vs.append(v)
        gs.append(g)
    v_out = np.empty((T, nc, n))
    s_out = np.empty((T, nc, n), dtype=bool)
    for t in range(T):
        ax = morph_axial(np.stack(vs), edges)
        for k, p in enumerate(params_list):
            cur = (i_series[t, k].reshape(n) + ax[k]).astype(dtype)
            v_new, g_new, spk = step(p, vs[k], gs[k], cur, step_index=t)
            vs[k], gs[k] = v_new, g_new
            v_out[t, k] = v_new
            s_out[t, k] = spk
    return v_out.reshape((T, nc) + shape), s_out.reshape((T, nc) + shape)
