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
