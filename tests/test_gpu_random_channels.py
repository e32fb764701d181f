"""Randomised custom channel tables (the north star's "custom channel
definitions"): the float64 kernels against the ORACLE (the restated reference,
dynamics.py:443-586 / adjoint.py:281-365) within 1e-9, and the NVRTC-generated
float32 kernels (merged form where its window proof holds, the direct step
elsewhere) under the per-neuron float32 contract against the oracle, every
failing neuron listed and attributed (tests/contract.py), none unexplained."""

import numpy as np
import pytest
import torch

from contract import check_against_oracle
from oracle import hh_oracle as O
from paper_2601_21407_b200 import _native as nat
from paper_2601_21407_b200 import adjoint as A
from paper_2601_21407_b200 import dynamics as Dy

pytestmark = pytest.mark.gpu


def _rate(rng, kind):
    v0 = rng.uniform(-70.0, -10.0)
    b = rng.choice([-1.0, 1.0]) * rng.uniform(4.0, 30.0)
    a = {"linoid": rng.uniform(0.01, 0.5), "exp": rng.uniform(0.005, 4.0),
         "sigmoid": rng.uniform(0.005, 4.0)}[kind]
    if kind == "linoid":
        a = abs(a) * np.sign(b)          # alpha > 0 for x / (1 - exp(-x / b))
    return Dy.RateFn(kind, float(a), float(v0), float(b))


def random_params(seed: int, dtype=np.float32):
    rng = np.random.default_rng(seed)
    if seed >= 12:   # tables the merged form cannot prove (a zero rate amplitude): the direct step
        base = random_params(seed - 12, dtype)
        ch = Dy.ChannelSpec("z", 0.5, -80.0, (Dy.GateSpec("c", Dy.RateFn("sigmoid", 0.0, -20.0, 5.0),
                                                          Dy.RateFn("exp", 0.005, -65.0, 40.0), 1),))
        return base.with_(channels=base.channels + (ch,))
    kinds = ["linoid", "exp", "sigmoid"]
    na = Dy.ChannelSpec("na", float(rng.uniform(40, 120)), 50.0, (
        Dy.GateSpec("m", _rate(rng, rng.choice(kinds)), _rate(rng, rng.choice(kinds)), 3),
        Dy.GateSpec("h", _rate(rng, "exp"), _rate(rng, "sigmoid"), 1)))
    k = Dy.ChannelSpec("k", float(rng.uniform(10, 40)), -90.0, (
        Dy.GateSpec("n", _rate(rng, rng.choice(kinds)), _rate(rng, rng.choice(kinds)), int(rng.integers(1, 5))),))
    chans = [na, k, Dy.ChannelSpec("leak", 0.3, -65.0)]
    if seed % 2:
        chans.append(Dy.ChannelSpec("x", float(rng.uniform(0.05, 2.0)), float(rng.uniform(-90, 120)), (
            Dy.GateSpec("q", _rate(rng, rng.choice(kinds)), _rate(rng, rng.choice(kinds)), 2),
            Dy.GateSpec("r", _rate(rng, rng.choice(kinds)), _rate(rng, rng.choice(kinds)), 1))))
    return Dy.HHParams(c_m=1.0, channels=tuple(chans), v_rest=-65.0, v_theta=0.0, dt=0.01,
                       rate_scale=float(rng.choice([1.0, 0.7, 2.0])), dtype=dtype)


@pytest.mark.parametrize("seed", list(range(12)) + [12, 15])
def test_random_channel_tables_forward_and_bptt(cuda, seed):
    p32 = random_params(seed)
    p64 = p32.with_(dtype=np.float64)
    rng = np.random.default_rng(100 + seed)
    n, T = 256, 400
    i = torch.as_tensor(rng.uniform(0.0, 15.0, size=(1, n)).repeat(T, 0), dtype=torch.float32, device=cuda)
    try:
        s0 = Dy.init_state(p64, (n,), device=cuda)
        tr64 = Dy.simulate(p64, i.double(), state0=s0)
    except Exception as e:   # a random table can blow up in float64 too: the same error in float32
        with pytest.raises(type(e)):
            Dy.simulate(p32, i, state0=Dy.init_state(p32, (n,), device=cuda))
        return
    ih = i.double().cpu().numpy()
    v_ref, s_ref = O.simulate(p64, ih)     # the float64 kernel ran it: the oracle must too
    v64 = tr64.v_series.double()
    assert np.array_equal(tr64.spike_series.cpu().numpy(), s_ref)
    err = np.abs(v64.cpu().numpy() - v_ref)
    assert np.all(err <= 1e-9 * np.abs(v_ref) + 1e-9), float(err.max())

    def ours(cols):
        tr = Dy.simulate(p32, torch.as_tensor(cols, dtype=torch.float32, device=cuda),
                         state0=Dy.init_state(p32, (cols.shape[1],), device=cuda))
        return tr.v_series.cpu().numpy(), tr.spike_series.cpu().numpy()

    v32, s32 = ours(ih)
    i_ext = np.concatenate([ih, ih[-2:]])          # the constant drive continues
    rep = check_against_oracle(p64, ih, v32, s32, v_ref, s_ref, ours_ext=ours, i_ext=i_ext)
    assert rep["unexplained"] == 0, [x for x in rep["listed"] if x["verdict"] == "unexplained"]
    # BPTT: d_i normwise within the 1e-3 contract (full storage)
    seed_v = 2.0 * v64 / v64.numel()
    r64 = A.backward_through_time(p64, Dy.init_state(p64, (n,), device=cuda), i.double(), seed_v)
    v0, g0 = O.rest_state(p64, n)
    ref = O.bptt(p64, v0, g0, ih, seed_v.cpu().numpy())
    d_i64 = r64.d_i.cpu().numpy()
    assert np.linalg.norm(d_i64 - ref["d_i"]) <= 1e-9 * np.linalg.norm(ref["d_i"])
    assert abs(r64.d_c_m - ref["d_c_m"]) <= 1e-9 * abs(ref["d_c_m"]) + 1e-15
    r32 = A.backward_through_time(p32, Dy.init_state(p32, (n,), device=cuda), i, seed_v.float())
    err = ((r32.d_i.double() - r64.d_i).norm() / r64.d_i.norm()).item()
    assert err < 1e-3, err
    assert abs(r32.d_c_m - r64.d_c_m) <= 1e-3 * abs(r64.d_c_m) + 1e-12


def test_random_tables_exercise_both_step_forms():
    """The random tables get the merged form; the zero-amplitude variants only
    the direct step."""
    assert all("// merged form off" not in nat.jit_source(random_params(s)) for s in range(12))
    assert all("// merged form off" in nat.jit_source(random_params(s)) for s in (12, 15))


def test_random_tables_spike(cuda):
    """The randomised tables are not all silent: most of them fire under the
    test's currents (so the spike-count checks above have something to check)."""
    firing = 0
    for seed in range(12):
        p = random_params(seed)
        n, T = 256, 400
        i = torch.as_tensor(np.random.default_rng(100 + seed).uniform(0.0, 15.0, size=(1, n)).repeat(T, 0),
                            dtype=torch.float32, device=cuda)
        try:
            tr = Dy.simulate(p, i, state0=Dy.init_state(p, (n,), device=cuda))
        except Exception:
            continue
        firing += int(tr.spike_series.any().item())
    assert firing >= 6, firing
