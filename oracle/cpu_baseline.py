"""Timed CPU baseline: the reference algorithm (restated in oracle/hh_oracle.py)
run on the host cores -- TEST/BENCH INFRASTRUCTURE ONLY.

Used by bench.py's `cpu_baseline` leg and its `--impl reference` arm, never
by the product.  P worker processes (one per host core, BLAS/OpenMP pinned to
1 thread) each run the reference's fused `hh_step` loop with a reused
workspace and ping-pong state buffers, recording V and spikes per step as
`simulate` does (dynamics.py:564-575), on a disjoint neuron shard -- the
concurrency the SPEC allows.  Imports numpy only (no torch), so
spawning many workers stays cheap.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time
from types import SimpleNamespace

import numpy as np


def _params_from_dict(d: dict, dtype) -> SimpleNamespace:
    chans = []
    for c in d["channels"]:
        gates = [SimpleNamespace(name=g["name"], exponent=int(g["exponent"]),
                                 alpha=SimpleNamespace(**g["alpha"]), beta=SimpleNamespace(**g["beta"]))
                 for g in c.get("gates", [])]
        chans.append(SimpleNamespace(name=c["name"], g_max=float(c["g_max"]), e_rev=float(c["e_rev"]),
                                     gates=tuple(gates)))
    return SimpleNamespace(c_m=d["c_m"], dt=d["dt"], v_rest=d["v_rest"], v_theta=d["v_theta"],
                           rate_scale=d["rate_scale"], channels=tuple(chans), dtype=dtype)


def _worker(args):
    pdict, dtype_name, n, seconds, min_steps, max_steps, seed, lam, amp = args
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    from oracle import hh_oracle as O
    dtype = np.dtype(dtype_name)
    p = _params_from_dict(pdict, dtype)
    rng = np.random.default_rng(seed)
    block = 16
    cur = (amp * rng.poisson(lam, size=(block, n))).astype(dtype)
    v, g = O.rest_state(p, n, dtype=dtype)
    sc = O.StepScratch(n, dtype)
    bufs = [(np.empty_like(v), np.empty_like(g)), (np.empty_like(v), np.empty_like(g))]
    vrec = np.empty((block, n), dtype=np.float64)
    srec = np.empty((block, n), dtype=bool)
    steps = 0
    t0 = time.perf_counter()
    while True:
        k = steps % block
        vo, go = bufs[steps % 2]
        v, g, sp = O.step(p, v, g, cur[k], sc, vo, go, step_index=steps)
        vrec[k] = v
        srec[k] = sp
        steps += 1
        el = time.perf_counter() - t0
        if steps >= max_steps or (steps >= min_steps and el >= seconds):
            break
    return n * steps, el


def run(params_dict: dict, dtype="float32", n_total: int = 1 << 21, seconds: float = 10.0,
        min_steps: int = 3, max_steps: int = 100000, workers: int | None = None, lam=2.0, amp=2.0):
    """Aggregate neuron-steps/s of `workers` processes on n_total neurons."""
    P = workers or os.cpu_count() or 1
    n_local = max(32, n_total // P)
    ctx = mp.get_context("spawn")
    jobs = [(params_dict, dtype, n_local, seconds, min_steps, max_steps, 1000 + r, lam, amp)
            for r in range(P)]
    with ctx.Pool(P) as pool:
        res = pool.map(_worker, jobs)
    ns = sum(r[0] for r in res)
    el = max(r[1] for r in res)
    return {"value": ns / el, "neuron_steps": ns, "seconds": el, "cores": P, "n_local": n_local,
            "steps_per_worker": [r[0] // n_local for r in res]}


# --------------------------------------------------------------------------- configs 3 / 4
def _worker_layers(args):
    """One core: the reference's readout composition (learn.py:238-274)
    generalised to a stack -- DenseLayer (x @ W.T + b, learn.py:210-211),
    simulate, then backward_through_time (adjoint.py:281-365, full storage,
    seed_spike from the next layer's dX) and the dW einsum (learn.py:272) --
    on batch-1 shards of the workload until `seconds` have elapsed.  Loss:
    MSE(V, 0) for one layer (config 3), cross-entropy on the time-mean output
    V for a stack (config 4).  Returns (neuron-steps through fwd + bwd, s)."""
    pdict, sizes, T, seconds, seed = args
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    from oracle import hh_oracle as O
    p = _params_from_dict(pdict, np.float64)
    rng = np.random.default_rng(seed)
    Ws = [rng.normal(0.05 if l == 0 else 0.02, 0.1 if l == 0 else 0.05, (sizes[l + 1], sizes[l]))
          for l in range(len(sizes) - 1)]
    per_sample = T * sum(sizes[1:])
    done = 0
    t0 = time.perf_counter()
    while True:
        x = ((rng.random((T, 1, sizes[0])) < 0.2) + 0.1 * rng.standard_normal((T, 1, sizes[0])))
        h, drives, ins, v = x, [], [], None
        for W in Ws:
            ins.append(h)
            d = O.dense(h, W, 0.0)
            v, s = O.simulate(p, d.reshape(T, -1))
            drives.append(d)
            h = s.reshape(T, 1, -1).astype(np.float64)
        if len(Ws) == 1:
            seed_v = 2.0 * v / v.size
        else:
            _, dl = O.cross_entropy_loss(v.reshape(T, 1, -1).mean(0), np.array([int(rng.integers(sizes[-1]))]))
            seed_v = np.broadcast_to(dl / T, (T, 1, sizes[-1])).reshape(T, -1)
        seed_s = None
        for l in range(len(Ws) - 1, -1, -1):
            n = sizes[l + 1]
            v0, g0 = O.rest_state(p, n)
            sv = seed_v if seed_v is not None else np.zeros((T, n))
            r = O.bptt(p, v0, g0, drives[l].reshape(T, -1), sv, seed_spike=seed_s)
            dd = r["d_i"].reshape(T, 1, n)
            O.dense_grad_w(dd.transpose(1, 0, 2), ins[l].transpose(1, 0, 2))
            seed_s = (dd @ Ws[l]).reshape(T, -1) if l > 0 else None
            seed_v = None
        done += per_sample
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done, el


def run_layers(params_dict: dict, sizes, T: int = 100, seconds: float = 10.0, workers: int | None = None):
    """Aggregate fwd + BPTT neuron-steps/s of `workers` processes (one per
    core), each on its own batch-1 shards of the config-3/4 workload (batch
    samples are independent: the reference's batch axis is data parallel)."""
    P = workers or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    jobs = [(params_dict, list(sizes), T, seconds, 2000 + r) for r in range(P)]
    with ctx.Pool(P) as pool:
        res = pool.map(_worker_layers, jobs)
    ns = sum(r[0] for r in res)
    el = max(r[1] for r in res)
    return {"value": ns / el, "neuron_steps": ns, "seconds": el, "cores": P,
            "samples": ns // (T * sum(sizes[1:]))}


# --------------------------------------------------------------------------- config 5
def run_network(params_dict: dict, offsets, targets, weights, delays, max_delay: int, lam, mu: float,
                sigma: float, psp_decay: float, steps: int = 200, warm: int = 100, seed: int = 0):
    """One core (network stepping is serial in the reference, cortex.py:379-438):
    `warm` + `steps` steps of step_network (cortex.py:273-310; oracle
    network_step) with the compound-Poisson background of cortex.py:225-232
    drawn by numpy; the last `steps` are timed.  Returns neuron-steps/s."""
    from oracle import hh_oracle as O
    p = _params_from_dict(params_dict, np.float64)
    n = len(offsets) - 1
    rng = np.random.default_rng(seed)
    v, g = O.rest_state(p, n)
    psp = np.zeros(n)
    ring = O.Ring(max_delay + 1, n)
    lam = np.asarray(lam, np.float64)
    t0 = None
    spikes = 0
    for t in range(warm + steps):
        if t == warm:
            t0 = time.perf_counter()
        k = rng.poisson(lam)
        bg = k * mu + sigma * np.sqrt(k) * rng.standard_normal(n)
        v, g, psp, sp = O.network_step(p, v, g, psp, ring, t, offsets, targets, weights, delays, psp_decay,
                                       background=bg)
        if t >= warm:
            spikes += int(sp.sum())
    el = time.perf_counter() - t0
    return {"value": n * steps / el, "seconds": el, "steps": steps, "cores": 1, "neurons": n,
            "spikes_per_step": spikes / steps}
