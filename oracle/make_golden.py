"""Generate the golden fixtures under tests/golden/ by RUNNING THE REFERENCE.

Test infrastructure only.  Imports the reference package `hhengine` from
/root/reference/pkg/src (read-only, present in the build container, NOT on
the GPU box) and records its outputs on small seeded cases.  The resulting
.npz files are committed; tests compare both the oracle restatement
(oracle/hh_oracle.py) and the CUDA product against them.

    python oracle/make_golden.py            # rewrites tests/golden/*.npz

Every case names the reference entry point it exercises.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF_SRC = os.environ.get("HH_REFERENCE_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import hhengine.adjoint as adj
    import hhengine.cortex as cortex
    import hhengine.defaults as defaults
    import hhengine.dynamics as dyn
    import hhengine.learn as learn
    import hhengine.reference as naive
    return dyn, adj, defaults, learn, cortex, naive


def _morph():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import hhengine.morphology as morph
    return morph


def c2_params(dyn, dt=0.01):
    """BASELINE config 2 custom set."""
    R, G, C = dyn.RateFn, dyn.GateSpec, dyn.ChannelSpec
    na = C("na", 50.0, 50.0, (
        G("m", R("linoid", 0.32, -43.2, 4.0), R("linoid", -0.28, -16.2, -5.0), 3),
        G("h", R("exp", 0.128, -39.2, 18.0), R("sigmoid", 4.0, -16.2, 5.0), 1)))
    kdr = C("k_dr", 5.0, -90.0, (
        G("n", R("linoid", 0.032, -41.2, 5.0), R("exp", 0.5, -46.2, 40.0), 4),))
    leak = C("leak", 0.0205, -70.3)
    cal = C("ca_l", 0.1, 120.0, (
        G("q", R("linoid", 0.055, -27.0, 3.8), R("exp", 0.94, -75.0, 17.0), 2),
        G("r", R("exp", 0.000457, -13.0, 50.0), R("sigmoid", 0.0065, -15.0, 28.0), 1)))
    kca = C("k_ca", 0.5, -90.0, (
        G("c", R("sigmoid", 0.01, -20.0, 5.0), R("exp", 0.005, -65.0, 40.0), 1),))
    return dyn.HHParams(c_m=1.0, channels=(na, kdr, leak, cal, kca), v_rest=-70.3,
                        v_theta=0.0, dt=dt)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    dyn, adj, defaults, learn, cortex, naive = _ref()
    os.makedirs(OUT, exist_ok=True)
    squid = defaults.squid_axon_params(dt=0.01)
    rs = defaults.cortical_rs_params(dt=0.1)
    c2 = c2_params(dyn)

    # -- known answers ----------
    ka = {}
    ka["gate_step"] = np.float64(dyn.gate_step(0.2, 0.5, 1.5, 0.1))
    st = dyn.NeuronState(np.array([-65.0]), np.zeros((0, 1)))
    ka["leak_current"] = dyn.ionic_current(st, (dyn.ChannelSpec("leak", 0.3, -54.4),))
    ka["spike_pairs"] = np.array([[-70, -69, 0], [-10, 10, 0], [0, 1, 0], [-1, 0, 0], [0, 0, 0]],
                                 dtype=np.float64)
    ka["spike_out"] = np.array([bool(dyn.spike_detect(a, b, c)) for a, b, c in ka["spike_pairs"]])
    plans = [(10, 10), (10, 20), (100, 10), (1, 5), (400, 20), (97, 7)]
    ka["plan_in"] = np.array(plans)
    ka["plan_seg"] = np.array([adj.make_plan(t, b).segment_length for t, b in plans])
    ka["plan_count"] = np.array([len(adj.make_plan(t, b).stored_indices) for t, b in plans])
    u = np.linspace(-40.0, 40.0, 161)
    ka["sur_u"] = u
    ka["sur_sig"] = adj.surrogate_grad(u, adj.SurrogateSpec("sigmoid-derivative", 2.5))
    ka["sur_rect"] = adj.surrogate_grad(u, adj.SurrogateSpec("rectangular", 2.5))
    ka["sur_default_squid"] = np.float64(adj.default_surrogate(defaults.squid_axon_params()).width)
    ka["sur_default_rs"] = np.float64(adj.default_surrogate(rs).width)
    for name, p in (("squid", squid), ("rs", rs), ("c2", c2)):
        vg = np.linspace(-120.0, 80.0, 401)
        sing = []
        for _, g in p.gate_layout:
            for fn in (g.alpha, g.beta):
                sing += [fn.v0, fn.v0 + 1e-9, fn.v0 - 1e-6, fn.v0 + 1e-3]
        vg = np.concatenate([vg, np.array(sing)])
        ka[f"{name}_vgrid"] = vg
        rows, slopes = [], []
        for _, g in p.gate_layout:
            a, b = dyn.gate_rates(g, vg, p.rate_scale)
            rows += [a, b]
            slopes += [g.alpha.deriv(vg), g.beta.deriv(vg)]
        ka[f"{name}_rates"] = np.array(rows)
        ka[f"{name}_slopes"] = np.array(slopes)
        ka[f"{name}_init_gates"] = dyn.init_state(p, (1,)).gates[:, 0]
        ka[f"{name}_init_gates_m55"] = dyn.init_state(p, (1,), v0=-55.0).gates[:, 0]
    # losses and their seeds (learn.py:80-107)
    rng_l = np.random.default_rng(5)
    lp, lt = rng_l.normal(size=(6, 4, 3)), rng_l.normal(size=(6, 4, 3))
    ka["mse_pred"], ka["mse_target"] = lp, lt
    ka["mse_loss"], ka["mse_seed"] = learn.mse_loss(lp, lt)
    ll, ly = 3.0 * rng_l.normal(size=(9, 10)), rng_l.integers(0, 10, size=9)
    ka["ce_logits"], ka["ce_target"] = ll, ly
    ka["ce_loss"], ka["ce_seed"] = learn.cross_entropy_loss(ll, ly)
    # multicompartment (morphology.py): coincidence demo, a random-current chain
    # with a batch axis, and axial_current of a random state
    morph = _morph()
    tr_demo = morph.coincidence_experiment(morph.coincidence_graph(), morph.demo_trials())
    chain = morph.chain_graph(5, defaults.squid_axon_params(dt=0.01), 0.5)
    rng_m = np.random.default_rng(7)
    i_chain = rng_m.uniform(0.0, 15.0, size=(300, 5, 3))
    tr_chain = morph.simulate_morphology(chain, i_chain)
    st_m = morph.init_morph_state(morph.coincidence_graph(), (4,))
    for k, s in enumerate(st_m.states):
        s.v[...] = rng_m.normal(-60.0, 8.0, size=4)
    ax_m = morph.axial_current(st_m, morph.coincidence_graph())
    np.savez_compressed(os.path.join(OUT, "morph.npz"),
                        demo_v0=tr_demo[0].v_series, demo_s0=tr_demo[0].spike_series,
                        demo_v1=tr_demo[1].v_series, demo_s1=tr_demo[1].spike_series,
                        chain_i=i_chain, chain_v=tr_chain.v_series, chain_s=tr_chain.spike_series,
                        ax_v=np.stack([s.v for s in st_m.states]), ax=ax_m)
    # run_network with a thalamic transient + SpikeRecord statistics (cortex.py:319-464)
    topo_t = cortex.build_network(0.02, 0, cortex.THALAMIC_CONFIG)
    thal = {"t_on_ms": 4.0, "duration_ms": 10.0, "rate_hz": 120.0, "weight": 0.22, "weight_std": 0.022}
    rec_t = cortex.run_network(topo_t, cortex.THALAMIC_CONFIG, 20.0, seed=3, warmup_ms=2.0, thalamic=thal)
    stats = {}
    for pop in ("L4e", "L2/3e", "L6i"):
        key = pop.replace("/", "")
        stats[f"rate_{key}"] = rec_t.pop_rate(pop)
        stats[f"quart_{key}"] = rec_t.rate_quartiles(pop)
        stats[f"cv_{key}"] = rec_t.isi_cv(pop)
        stats[f"hist_{key}"] = rec_t.rate_histogram(pop, 2.0)[1]
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        fn = os.path.join(td, "r.ndjson")
        rec_t.to_ndjson(fn)
        nd = open(fn).read()
    np.savez_compressed(os.path.join(OUT, "cortex_thalamic.npz"), spike_t=rec_t.times_ms, spike_id=rec_t.neuron_ids,
                        ndjson=np.array(nd), **stats)
    # LIF baseline (dynamics.py:532-586 LIF branch, adjoint.py:197-227)
    lifp = defaults.lif_params()
    rng_l2 = np.random.default_rng(11)
    i_lif = rng_l2.uniform(0.0, 2.5, size=(400, 6))
    tr_lif = dyn.simulate(lifp, i_lif)
    tr_lif32 = dyn.simulate(lifp.__class__(lifp.tau, lifp.v_theta, lifp.v_reset, lifp.dt, np.float32),
                            i_lif.astype(np.float32))
    st_l = dyn.NeuronState(rng_l2.uniform(0.0, 1.2, size=6), np.zeros((0, 6)))
    adj_o = adj.AdjointState(rng_l2.normal(size=6), np.zeros((0, 6)), 0.0, np.zeros(0),
                             d_spike=rng_l2.normal(size=6))
    sur_l = adj.default_surrogate(lifp)
    a_in, d_i_l = adj.lif_step_backward(st_l, i_lif[0], lifp, adj_o, sur_l)
    adj_o2 = adj.AdjointState(adj_o.d_v, np.zeros((0, 6)), 0.0, np.zeros(0))
    a_in2, d_i_l2 = adj.lif_step_backward(st_l, i_lif[0], lifp, adj_o2, sur_l)
    np.savez_compressed(os.path.join(OUT, "lif.npz"), i=i_lif, v=tr_lif.v_series, s=tr_lif.spike_series,
                        v32=tr_lif32.v_series, s32=tr_lif32.spike_series, st_v=st_l.v, d_v=adj_o.d_v,
                        d_spike=adj_o.d_spike, sur_w=sur_l.width, bwd_dv=a_in.d_v, bwd_di=d_i_l,
                        bwd2_dv=a_in2.d_v, bwd2_di=d_i_l2)
    # training plumbing (learn.py:33-151): psp_filter, smape, adam_step
    kern = learn.PSPKernel(2.0, 12, 0.1)
    rng_p = np.random.default_rng(13)
    sp_in = (rng_p.random((80, 3, 7)) < 0.2).astype(np.float64) + 0.05 * rng_p.normal(size=(80, 3, 7))
    ka["psp_in"], ka["psp_out"] = sp_in, learn.psp_filter(sp_in, kern)
    ka["smape_a"], ka["smape_b"] = rng_p.normal(size=40), rng_p.normal(size=40)
    ka["smape_a"][3] = ka["smape_b"][3] = 0.0
    ka["smape"] = learn.smape(ka["smape_a"], ka["smape_b"])
    st_a = learn.AdamState(lr=1e-2)
    pa = {"w": rng_p.normal(size=(4, 3)), "b": rng_p.normal(size=3)}
    ka["adam_w0"], ka["adam_b0"] = pa["w"].copy(), pa["b"].copy()
    gs = []
    for k in range(3):
        gr = {"w": rng_p.normal(size=(4, 3)), "b": rng_p.normal(size=3)}
        gs.append(gr)
        pa = learn.adam_step(pa, gr, st_a, lr=learn.cosine_lr(1e-2, k, 3))
    ka["adam_gw"] = np.stack([g["w"] for g in gs])
    ka["adam_gb"] = np.stack([g["b"] for g in gs])
    ka["adam_w3"], ka["adam_b3"] = pa["w"], pa["b"]
    # rest-state population rates at scale 0.1 (cortex.py:441-448), the
    # statistical target of the device-background runs
    rec_r = cortex.rest_state_run(1200.0, 0.1, 0, warmup_ms=200.0)
    ka["rest_rates"] = np.array([rec_r.pop_rate(p.name) for p in rec_r.topo.populations])
    # the step-level background draw (cortex.py:225-232)
    ka["bg_lam"] = np.linspace(0.0, 3.0, 40)
    ka["bg_sample"] = cortex.background_sample(ka["bg_lam"], 0.11, 0.02, 40, np.random.default_rng(21))
    np.savez_compressed(os.path.join(OUT, "known_answers.npz"), **ka)

    # -- forward traces (dynamics.simulate / reference.naive_simulate) -------
    n = 32
    i_ramp = np.tile(20.0 * np.arange(n) / (n - 1), (2000, 1))
    tr, fin = dyn.simulate(squid, i_ramp, record_state=True)
    tr_naive = naive.naive_simulate(squid, i_ramp)
    assert np.array_equal(tr.v_series, tr_naive.v_series)
    np.savez_compressed(os.path.join(OUT, "fwd_squid_ramp.npz"), i=i_ramp[0], T=2000,
                        v=tr.v_series, spikes=tr.spike_series, v_fin=fin.v, g_fin=fin.gates)

    # config 1 on one neuron, full 10,000-step horizon (all 1,024 neurons are identical)
    i1 = np.full((10000, 1), 10.0)
    tr1 = dyn.simulate(squid, i1)
    # the reference's own float32 mode on the same case (hh_step loop, dynamics.py:176)
    p32 = squid.with_(dtype=np.float32)
    s32 = dyn.init_state(p32, (1,))
    v32 = np.empty((10000, 1), dtype=np.float32)
    k32 = np.empty((10000, 1), dtype=bool)
    for t in range(10000):
        s32, sp = dyn.hh_step(s32, i1[t], p32, step_index=t)
        v32[t], k32[t] = s32.v, sp
    np.savez_compressed(os.path.join(OUT, "fwd_c1_one.npz"), v=tr1.v_series[:, 0],
                        spikes=tr1.spike_series[:, 0], v32=v32[:, 0], spikes32=k32[:, 0])

    rng = np.random.default_rng(7)
    i_rs = rng.normal(8.0, 3.0, size=(600, 16))
    tr_rs = dyn.simulate(rs, i_rs)
    np.savez_compressed(os.path.join(OUT, "fwd_rs.npz"), i=i_rs, v=tr_rs.v_series,
                        spikes=tr_rs.spike_series)

    i_c2 = 2.0 * np.random.default_rng(0).poisson(2.0, size=(1500, 16)).astype(np.float64)
    tr_c2, fin2 = dyn.simulate(c2, i_c2, record_state=True)
    np.savez_compressed(os.path.join(OUT, "fwd_c2.npz"), i=i_c2, v=tr_c2.v_series,
                        spikes=tr_c2.spike_series, v_fin=fin2.v, g_fin=fin2.gates,
                        params=np.array([repr(c2.to_dict())]))

    # rate_scale + non-rest start + scalar current through hh_step directly
    sc = defaults.squid_axon_params(dt=0.025, rate_scale=1.7)
    s0 = dyn.init_state(sc, (8,), v0=-60.0)
    s0.v = s0.v + np.linspace(-3.0, 3.0, 8)
    vv, ss = [], []
    st = s0
    for t in range(400):
        st, sp = dyn.hh_step(st, 14.0, sc, step_index=t)
        vv.append(st.v.copy())
        ss.append(sp)
    np.savez_compressed(os.path.join(OUT, "fwd_scaled_scalar.npz"), v0=s0.v, g0=s0.gates,
                        v=np.array(vv), spikes=np.array(ss))

    # -- gradients (adjoint.backward_through_time / hh_step_backward) -------
    def bptt_case(fname, p, n, T, mean, std, seed, sur=None, budget=7):
        r = np.random.default_rng(seed)
        i_s = r.normal(mean, std, size=(T, n))
        s0 = dyn.init_state(p, (n,))
        seed_v = r.normal(0.0, 1.0, size=(T, n)) * 0.01
        seed_sp = r.normal(0.0, 1.0, size=(T, n))
        full = adj.backward_through_time(p, s0, i_s, seed_v, seed_sp, surrogate=sur)
        pl = adj.backward_through_time(p, s0, i_s, seed_v, seed_sp,
                                       plan=adj.make_plan(T, budget), surrogate=sur)
        nos = adj.backward_through_time(p, s0, i_s, seed_v, None, surrogate=sur)
        tr = dyn.simulate(p, i_s)
        np.savez_compressed(
            os.path.join(OUT, fname), i=i_s, seed_v=seed_v, seed_spike=seed_sp,
            spikes=tr.spike_series, v=tr.v_series,
            d_i=full.d_i, d_v0=full.d_state0.d_v, d_g0=full.d_state0.d_gates,
            d_c_m=np.float64(full.d_c_m), d_g_max=full.d_g_max,
            plan_d_i=pl.d_i, plan_d_c_m=np.float64(pl.d_c_m), plan_d_g_max=pl.d_g_max,
            plan_calls=pl.stats.forward_calls, plan_peak=pl.stats.peak_stored_states,
            full_calls=full.stats.forward_calls, full_peak=full.stats.peak_stored_states,
            nos_d_i=nos.d_i, nos_d_c_m=np.float64(nos.d_c_m), nos_d_g_max=nos.d_g_max,
            budget=budget, sur=np.array([sur.kind, sur.width] if sur else ["", 0.0]))

    bptt_case("bptt_rs.npz", rs, 8, 60, 9.0, 4.0, 11)
    bptt_case("bptt_squid_rect.npz", defaults.squid_axon_params(dt=0.025, rate_scale=1.3),
              6, 80, 9.0, 5.0, 12, sur=adj.SurrogateSpec("rectangular", 3.0))
    bptt_case("bptt_c2.npz", c2_params(dyn, dt=0.02), 5, 160, 30.0, 6.0, 13, budget=9)

    r = np.random.default_rng(21)
    nst = 10
    s_in = dyn.init_state(c2, (nst,), v0=-50.0)
    s_in.v = r.uniform(-80.0, 30.0, nst)
    s_in.gates = r.uniform(0.0, 1.0, s_in.gates.shape)
    ao = adj.AdjointState(d_v=r.normal(size=nst), d_gates=r.normal(size=s_in.gates.shape),
                          d_c_m=0.25, d_g_max=r.normal(size=len(c2.channels)),
                          d_spike=r.normal(size=nst))
    i_in = r.normal(5.0, 2.0, nst)
    sur = adj.default_surrogate(c2)
    ai, di = adj.hh_step_backward(s_in, i_in, c2, ao, sur, step_index=3)
    np.savez_compressed(os.path.join(OUT, "step_backward_c2.npz"), v=s_in.v, g=s_in.gates,
                        i=i_in, d_v=ao.d_v, d_g=ao.d_gates, d_c_m_in=np.float64(ao.d_c_m),
                        d_g_max_in=ao.d_g_max, d_spike=ao.d_spike, out_d_v=ai.d_v,
                        out_d_g=ai.d_gates, out_d_c_m=np.float64(ai.d_c_m),
                        out_d_g_max=ai.d_g_max, out_d_i=di)

    # -- dense projection -> simulate -> BPTT -> dW (learn.py:238-274 generalised)
    r = np.random.default_rng(3)
    B, T, C, O = 3, 25, 12, 5
    x = (r.random((B, T, C)) < 0.3).astype(np.float64) + 0.1 * r.normal(size=(B, T, C))
    w = r.normal(3.0, 1.0, size=(O, C))
    b = r.normal(0.5, 0.2, size=O)
    layer = learn.DenseLayer(w, b)
    drive = layer(x)                                   # (B, T, O)
    i_s = np.ascontiguousarray(np.moveaxis(drive, 0, 1))  # (T, B, O)
    tr = dyn.simulate(rs, i_s)
    loss, seed = learn.mse_loss(tr.v_series, np.zeros_like(tr.v_series))
    res = adj.backward_through_time(rs, dyn.init_state(rs, (B, O)), i_s, seed)
    d_drive = np.moveaxis(res.d_i, 0, 1)               # (B, T, O)
    d_w = np.einsum("btc,btk->ck", d_drive, x)
    np.savez_compressed(os.path.join(OUT, "readout_rs.npz"), x=x, w=w, b=b, v=tr.v_series,
                        spikes=tr.spike_series, loss=np.float64(loss), d_i=res.d_i, d_w=d_w,
                        d_b=d_drive.sum(axis=(0, 1)), d_c_m=np.float64(res.d_c_m),
                        d_g_max=res.d_g_max)

    # -- teacher-student readout fitting (learn.py:223-377) -------------------
    task = learn.make_teacher_student_task(n_channels=16, n_steps=120, n_train=4, n_val=3, pad_len=20, seed=2)
    student = learn.make_student(task, seed=5)
    w_init = student.dense.weights.copy()
    filt = task.teacher.filter_inputs(task.train_inputs)
    pred_t, v_t = task.teacher.forward(filt)
    rng_g = np.random.default_rng(17)
    seed_pred = rng_g.normal(size=pred_t.shape) * 1e-2
    g_t = task.teacher.grads(filt, seed_pred, v_t)
    hist = learn.fit(student, task, learn.TrainConfig(epochs=5, lr=2e-2))
    seg = learn.segment_traces(np.arange(50.0), 2.0 * np.arange(50.0), learn.SegmentationScheme(7, 9))
    tr_idx, te_idx = learn.split_dataset(11, np.random.default_rng(4))
    np.savez_compressed(os.path.join(OUT, "readout_fit.npz"),
                        train_inputs=task.train_inputs, train_targets=task.train_targets,
                        val_inputs=task.val_inputs, val_targets=task.val_targets,
                        teacher_w=task.teacher.dense.weights, filtered=filt, teacher_v=v_t,
                        seed_pred=seed_pred, g_w=g_t["w"], g_b=g_t["b"], g_sw=np.float64(g_t["scale_w"]),
                        g_sb=np.float64(g_t["scale_b"]), student_w0=w_init, history=np.array(hist),
                        final_w=student.dense.weights, final_b=student.dense.bias,
                        final_sw=np.float64(student.scale_w), final_sb=np.float64(student.scale_b),
                        seg_in=np.array([a for a, _ in seg]), seg_out=np.array([b for _, b in seg]),
                        split_train=tr_idx, split_test=te_idx)

    # -- cortex topology + short network run (cortex.py:138-218, :379-438) ---
    topo = cortex.build_network(0.02, 0)
    rec = cortex.run_network(topo, cortex.REST_CONFIG, 20.0, seed=1)
    np.savez_compressed(
        os.path.join(OUT, "cortex_small.npz"), scale=0.02, seed=0, run_seed=1, duration_ms=20.0,
        n_neurons=topo.n_neurons, n_synapses=topo.n_synapses, max_delay=topo.max_delay,
        sizes=np.array([p.size for p in topo.populations]),
        sha_offsets=_sha(topo.syn_offsets), sha_target=_sha(topo.syn_target),
        sha_weight=_sha(topo.syn_weight), sha_delay=_sha(topo.syn_delay),
        head_target=topo.syn_target[:200], head_weight=topo.syn_weight[:200],
        head_delay=topo.syn_delay[:200], offsets=topo.syn_offsets,
        spike_t=rec.times_ms, spike_id=rec.neuron_ids)
    # the reference's public API per module (names the drop-in must provide)
    import importlib
    import json
    api = {}
    for m in ("dynamics", "adjoint", "defaults", "errors", "learn", "morphology", "connectivity", "reference",
              "cortex"):
        mod = importlib.import_module("hhengine." + m)
        names = {n for n in dir(mod) if not n.startswith("_")
                 and getattr(getattr(mod, n), "__module__", None) == "hhengine." + m}
        names |= {n for n in dir(mod) if n.isupper() and not n.startswith("_")}
        api[m] = sorted(names)
    with open(os.path.join(OUT, "api_names.json"), "w") as f:
        json.dump(api, f, indent=1, sort_keys=True)
    print("golden fixtures written to", os.path.abspath(OUT))


if __name__ == "__main__":
    main()
