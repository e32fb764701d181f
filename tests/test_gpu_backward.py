"""GPU parity of the gradient path (hhb_backward) against the reference's
golden BPTT vectors, finite differences and its own plan invariance.

Tolerances:
  float64 build: d_i, d_state0, d_c_m, d_g_max within 1e-9 relative (normwise)
                 of the reference.
  float32 build: d_i normwise rel <= 1e-3, d_c_m / d_g_max rel <= 1e-3 against
                 the float64 reference.
  plan invariance: bit-exact for any checkpoint spacing.
"""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import hh_oracle as O
from paper_2601_21407_b200 import adjoint as A
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200 import dynamics as Dy
from paper_2601_21407_b200.errors import GradientOverflowError, UsageError

pytestmark = pytest.mark.gpu


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


CASES = {
    "bptt_rs": lambda: DF.cortical_rs_params(dt=0.1),
    "bptt_squid_rect": lambda: DF.squid_axon_params(dt=0.025, rate_scale=1.3),
    "bptt_c2": lambda: DF.na_kdr_cal_kca_params(dt=0.02),
}


def _sur(g):
    kind, width = str(g["sur"][0]), float(g["sur"][1])
    return A.SurrogateSpec(kind, width) if kind else None


@pytest.mark.parametrize("case", list(CASES))
def test_fp64_bptt_matches_reference(cuda, case):
    g = golden(case)
    p = CASES[case]()
    n = g["i"].shape[1]
    s0 = Dy.init_state(p, (n,))
    T = g["i"].shape[0]
    full = A.backward_through_time(p, s0, g["i"], g["seed_v"], g["seed_spike"], surrogate=_sur(g))
    assert nrel(full.d_i, g["d_i"]) < 1e-9
    assert nrel(full.d_state0.d_v, g["d_v0"]) < 1e-9
    assert nrel(full.d_state0.d_gates, g["d_g0"]) < 1e-9
    assert abs(full.d_c_m - float(g["d_c_m"])) <= 1e-9 * abs(float(g["d_c_m"]))
    assert nrel(full.d_g_max, g["d_g_max"]) < 1e-9
    assert (full.stats.forward_calls, full.stats.peak_stored_states) == (int(g["full_calls"]), int(g["full_peak"]))
    plan = A.make_plan(T, int(g["budget"]))
    pl = A.backward_through_time(p, s0, g["i"], g["seed_v"], g["seed_spike"], plan=plan, surrogate=_sur(g))
    assert nrel(pl.d_i, g["plan_d_i"]) < 1e-9
    assert (pl.stats.forward_calls, pl.stats.peak_stored_states) == (int(g["plan_calls"]), int(g["plan_peak"]))
    nos = A.backward_through_time(p, s0, g["i"], g["seed_v"], None, surrogate=_sur(g))
    assert nrel(nos.d_i, g["nos_d_i"]) < 1e-9
    assert nrel(nos.d_g_max, g["nos_d_g_max"]) < 1e-9


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_plan_invariance_is_bit_exact(cuda, dtype):
    p = DF.na_kdr_cal_kca_params(dt=0.02).with_(dtype=dtype)
    rng = np.random.default_rng(4)
    T, n = 97, 300
    i = rng.normal(25, 8, size=(T, n))
    sv = rng.normal(0, 0.01, size=(T, n))
    ss = rng.normal(0, 1, size=(T, n))
    s0 = Dy.init_state(p, (n,))
    ref = A.backward_through_time(p, s0, i, sv, ss)
    for budget in (1, 5, 13, 97):
        r = A.backward_through_time(p, s0, i, sv, ss, plan=A.make_plan(T, budget))
        assert np.array_equal(r.d_i, ref.d_i), budget
        assert np.array_equal(r.d_state0.d_gates, ref.d_state0.d_gates)
        assert r.d_c_m == ref.d_c_m and np.array_equal(r.d_g_max, ref.d_g_max)


@pytest.mark.parametrize("case", list(CASES))
def test_fp32_bptt_contract(cuda, case):
    g = golden(case)
    p = CASES[case]().with_(dtype=np.float32)
    n = g["i"].shape[1]
    r = A.backward_through_time(p, Dy.init_state(p, (n,)), g["i"], g["seed_v"], g["seed_spike"],
                                surrogate=_sur(g))
    # spikes of the fp32 forward must match the reference for the pointwise
    # comparison to be meaningful; the normwise bound is the contract
    assert nrel(r.d_i, g["d_i"]) < 1e-3
    assert abs(r.d_c_m - float(g["d_c_m"])) <= 1e-3 * abs(float(g["d_c_m"]))
    assert nrel(r.d_g_max, g["d_g_max"]) < 1e-3


def test_fp64_step_backward_matches_reference(cuda):
    g = golden("step_backward_c2")
    p = DF.na_kdr_cal_kca_params()
    adj = A.AdjointState(g["d_v"], g["d_g"], float(g["d_c_m_in"]), g["d_g_max_in"], g["d_spike"])
    ai, di = A.hh_step_backward(Dy.NeuronState(g["v"], g["g"]), g["i"], p, adj,
                                A.default_surrogate(p), step_index=3)
    assert nrel(ai.d_v, g["out_d_v"]) < 1e-12
    assert nrel(ai.d_gates, g["out_d_g"]) < 1e-12
    assert nrel(di, g["out_d_i"]) < 1e-12
    assert abs(ai.d_c_m - float(g["out_d_c_m"])) < 1e-12 * abs(float(g["out_d_c_m"]))
    assert nrel(ai.d_g_max, g["out_d_g_max"]) < 1e-12


def test_finite_differences_fp64(cuda):
    """loss = sum V over a 50-step chain, d_i and d_c_m / d_g_max
    against central differences (h=1e-5) within 1e-5 relative."""
    p = DF.cortical_rs_params(dt=0.05)
    rng = np.random.default_rng(2)
    T, n = 50, 6
    i = rng.normal(6, 2, size=(T, n))
    s0 = Dy.init_state(p, (n,))
    res = A.backward_through_time(p, s0, i, np.ones((T, n)))

    base = Dy.simulate(p, i, state0=s0).v_series

    def loss(ii, q=p):
        # sum(V - V_base): same gradient as sum(V), without the cancellation
        # of two ~2e4 totals that would swamp a central difference at h=1e-5
        return float((Dy.simulate(q, ii, state0=s0).v_series - base).sum())

    h = 1e-5
    for (t, j) in [(0, 0), (10, 3), (25, 5), (49, 1)]:
        ip, im = i.copy(), i.copy()
        ip[t, j] += h
        im[t, j] -= h
        fd = (loss(ip) - loss(im)) / (2 * h)
        assert abs(res.d_i[t, j] - fd) <= 1e-5 * abs(fd) + 1e-8
    fd_cm = (loss(i, p.with_(c_m=p.c_m + h)) - loss(i, p.with_(c_m=p.c_m - h))) / (2 * h)
    assert abs(res.d_c_m - fd_cm) <= 1e-5 * abs(fd_cm) + 1e-8
    # the leak gradient is ~3e-3; at h=1e-5 the summed V rounding (~300 x 1e-14)
    # is ~1e-7 of FD noise, so the g_max differences use h=1e-4 (truncation ~h^2)
    hg = 1e-4
    for ci, ch in enumerate(p.channels):
        def with_g(dg):
            chans = list(p.channels)
            chans[ci] = Dy.ChannelSpec(ch.name, ch.g_max + dg, ch.e_rev, ch.gates)
            return p.with_(channels=tuple(chans))
        fd_g = (loss(i, with_g(hg)) - loss(i, with_g(-hg))) / (2 * hg)
        assert abs(res.d_g_max[ci] - fd_g) <= 1e-5 * abs(fd_g) + 1e-8


def test_zero_seed_gives_zero_gradient_and_usage_errors(cuda):
    p = DF.squid_axon_params(dt=0.02)
    i = np.full((30, 4), 12.0)
    s0 = Dy.init_state(p, (4,))
    r = A.backward_through_time(p, s0, i, np.zeros((30, 4)))
    assert not np.any(r.d_i) and r.d_c_m == 0.0 and not np.any(r.d_g_max)
    with pytest.raises(UsageError):
        A.backward_through_time(p, s0, i, np.zeros((29, 4)))
    with pytest.raises(UsageError):
        A.backward_through_time(p, s0, i, np.zeros((30, 4)), plan=A.make_plan(31, 3))


def test_zero_conductance_dv_di(cuda):
    """zero-conductance neuron, d(V')/d(i_ext) = dt/c_m exactly."""
    p = DF.squid_axon_params(g_na=0.0, g_k=0.0, g_leak=0.0, dt=0.05, c_m=2.0)
    s0 = Dy.init_state(p, (3,))
    adj = A.AdjointState(np.ones(3), np.zeros((3, 3)), 0.0, np.zeros(3))
    _, di = A.hh_step_backward(s0, 1.0, p, adj, A.default_surrogate(p))
    assert np.all(di == 0.05 / 2.0)


def test_gradient_overflow_step_index(cuda):
    p = DF.squid_axon_params(dt=0.02)
    T, n = 40, 8
    i = np.full((T, n), 8.0)
    sv = np.zeros((T, n))
    sv[23, 5] = 1e308
    sv[22, 5] = 1e308
    with pytest.raises(GradientOverflowError) as e:
        A.backward_through_time(p, Dy.init_state(p, (n,)), i, sv * 10)
    assert e.value.step_index in (22, 23)


def test_readout_layer_composition_fp64(cuda):
    """dense -> simulate -> BPTT -> dW (learn.py:238-274 generalised) on device."""
    g = golden("readout_rs")
    p = DF.cortical_rs_params(dt=0.1)
    drive = g["x"] @ g["w"].T + g["b"]
    i_s = np.ascontiguousarray(np.moveaxis(drive, 0, 1))
    tr = Dy.simulate(p, i_s)
    assert nrel(tr.v_series, g["v"]) < 1e-12
    seed = 2.0 * tr.v_series / tr.v_series.size
    res = A.backward_through_time(p, Dy.init_state(p, i_s.shape[1:]), i_s, seed)
    assert nrel(res.d_i, g["d_i"]) < 1e-9
    d_w = np.einsum("btc,btk->ck", np.moveaxis(res.d_i, 0, 1), g["x"])
    assert nrel(d_w, g["d_w"]) < 1e-9


def test_device_tensors_path(cuda):
    p = DF.cortical_rs_params(dt=0.1).with_(dtype=np.float32)
    rng = np.random.default_rng(8)
    i = torch.tensor(rng.normal(9, 3, size=(60, 500)), dtype=torch.float32, device=cuda)
    sv = torch.tensor(rng.normal(0, 0.01, size=(60, 500)), dtype=torch.float32, device=cuda)
    s0 = Dy.init_state(p, (500,), device=cuda)
    r = A.backward_through_time(p, s0, i, sv, plan=A.make_plan(60, 6))
    assert isinstance(r.d_i, torch.Tensor) and r.d_i.is_cuda and r.d_i.dtype == torch.float32
    r2 = A.backward_through_time(p, s0, i.cpu().numpy(), sv.cpu().numpy(), plan=A.make_plan(60, 6))
    assert np.array_equal(r.d_i.cpu().numpy(), r2.d_i.astype(np.float32))


def _fd_chains(cuda, p, n, T, rng, h=2e-5, hp=2e-5):
    """n independent chains (one neuron each) of one parameter set: random
    drive and random membrane-potential loss L_j = sum_t w[t, j] V[t, j].
    Central differences with one Richardson step, (4 D(h/2) - D(h)) / 3
    (truncation O(h^4): the spike upstroke makes V strongly nonlinear in
    I and the parameters); each difference sums w (V+ - V-) elementwise."""
    mu = rng.uniform(0.0, 15.0, size=n)
    i = rng.normal(mu, 3.0, size=(T, n))
    w = rng.normal(0.0, 1.0, size=(T, n))
    it = torch.as_tensor(i, device=cuda)
    res = A.backward_through_time(p, Dy.init_state(p, (n,), device=cuda), it, torch.as_tensor(w, device=cuda))
    d_i = res.d_i.cpu().numpy()

    def v_of(ii, q=p):
        return Dy.simulate(q, torch.as_tensor(ii, device=cuda), state0=Dy.init_state(q, (n,), device=cuda)) \
            .v_series.cpu().numpy()

    errs = []
    # d_i at three random steps per chain, all chains at once (chains are independent)
    for _ in range(3):
        ts = rng.integers(0, T, size=n)
        def d(hh):
            ip, im = i.copy(), i.copy()
            ip[ts, np.arange(n)] += hh
            im[ts, np.arange(n)] -= hh
            return (w * (v_of(ip) - v_of(im))).sum(0) / (2 * hh)
        fd = (4 * d(h / 2) - d(h)) / 3
        ad = d_i[ts, np.arange(n)]
        floor = 1e-6 * np.abs(d_i).max(0)
        errs.append(np.abs(ad - fd) / np.maximum(np.abs(fd), floor))
        print("d_i", p.channels[0].name, float(errs[-1].max()))
    # parameter gradients are population sums: one adjoint run per chain.
    # They are compared as one vector per chain in log-parameter space,
    # u = (c_m dL/dc_m, g_1 dL/dg_1, ...), normwise: a channel that barely
    # conducts has dL/dg ~ 1e-7 of the others, below the central difference's
    # rounding noise, so an elementwise relative error there measures the FD
    # noise, not the adjoint
    d_cm = np.empty(n)
    d_gm = np.empty((n, len(p.channels)))
    for j in range(n):
        r = A.backward_through_time(p, Dy.init_state(p, (1,), device=cuda), it[:, j:j + 1],
                                    torch.as_tensor(w[:, j:j + 1], device=cuda))
        d_cm[j] = r.d_c_m
        d_gm[j] = np.asarray(r.d_g_max)

    def rich(q_of):
        def d(hh):
            return (w * (v_of(i, q_of(hh)) - v_of(i, q_of(-hh)))).sum(0) / (2 * hh)
        return (4 * d(hp / 2) - d(hp)) / 3

    u_fd = [rich(lambda dh: p.with_(c_m=p.c_m * (1 + dh)))]
    u_ad = [p.c_m * d_cm]
    for ci, ch in enumerate(p.channels):
        def with_g(dh, ci=ci, ch=ch):
            chans = list(p.channels)
            chans[ci] = Dy.ChannelSpec(ch.name, ch.g_max * (1 + dh), ch.e_rev, ch.gates)
            return p.with_(channels=tuple(chans))
        u_fd.append(rich(with_g))
        u_ad.append(ch.g_max * d_gm[:, ci])
    u_fd, u_ad = np.stack(u_fd, 1), np.stack(u_ad, 1)
    errs.append(np.linalg.norm(u_ad - u_fd, axis=1) / np.linalg.norm(u_fd, axis=1))
    print("params", p.channels[0].name, float(errs[-1].max()))
    return np.concatenate(errs)


def test_spec_acceptance1_fd_over_120_random_chains(cuda):
    """SPEC.md:569 acceptance 1: over >= 100 random HH chains (T <= 100,
    float64) the adjoint gradients match central finite differences within
    1e-5 relative for membrane-potential losses.  120 chains = 40 each of the
    squid, RS and config-2 parameter sets with random drive and random loss
    weights; per chain d_i at 3 random steps (relative to max(|FD|, 1e-6 x the
    chain's largest d_i)) and the parameter gradients d_c_m, d_g_max as one
    log-parameter vector (normwise; see _fd_chains)."""
    rng = np.random.default_rng(11)
    errs = []
    for p in (DF.squid_axon_params(dt=0.02), DF.cortical_rs_params(dt=0.05), DF.na_kdr_cal_kca_params(dt=0.02)):
        errs.append(_fd_chains(cuda, p, 40, 100, rng))
    e = np.concatenate(errs)
    assert e.size >= 120 * 4
    print("FD max rel err", float(e.max()), "p99", float(np.quantile(e, 0.99)))
    assert e.max() < 1e-5, float(e.max())
