"""Pin the CPU oracle (oracle/hh_oracle.py) to the reference's own outputs.

The golden vectors were produced by running the reference package in the
build container (oracle/make_golden.py).  The oracle restates the same NumPy
operation order, so most checks are bit-exact.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import hh_oracle as O
from paper_2601_21407_b200 import defaults as DF


def _sets():
    return {"squid": DF.squid_axon_params(dt=0.01), "rs": DF.cortical_rs_params(dt=0.1),
            "c2": DF.na_kdr_cal_kca_params(dt=0.01)}


def test_known_answers():
    ka = golden("known_answers")
    # SPEC.md:81 gate_step(p=0.2, a=0.5, b=1.5, dt=0.1)
    assert float(ka["gate_step"]) == 0.25 + (0.2 - 0.25) * np.exp(-0.2)
    assert np.allclose(ka["leak_current"], -3.18, rtol=0, atol=1e-12)
    assert [bool(x) for x in ka["spike_out"]] == [False, True, False, True, False]
    for (T, b), seg, cnt in zip(ka["plan_in"], ka["plan_seg"], ka["plan_count"]):
        s, idx = O.plan(int(T), int(b))
        assert s == seg and len(idx) == cnt
    u = ka["sur_u"]
    assert np.array_equal(O.surrogate(u, "sigmoid-derivative", 2.5), ka["sur_sig"])
    assert np.array_equal(O.surrogate(u, "rectangular", 2.5), ka["sur_rect"])
    assert O.default_width(DF.squid_axon_params()) == float(ka["sur_default_squid"]) == 16.25
    assert O.default_width(DF.cortical_rs_params()) == float(ka["sur_default_rs"])


@pytest.mark.parametrize("name", ["squid", "rs", "c2"])
def test_rates_slopes_init(name):
    ka = golden("known_answers")
    p = _sets()[name]
    vg = ka[f"{name}_vgrid"]
    rows, slopes = [], []
    for _, g in O.gate_list(p):
        rows += [O.rate_value(g.alpha, vg), O.rate_value(g.beta, vg)]
        slopes += [O.rate_slope(g.alpha, vg), O.rate_slope(g.beta, vg)]
    assert np.array_equal(np.array(rows), ka[f"{name}_rates"])
    assert np.array_equal(np.array(slopes), ka[f"{name}_slopes"])
    assert np.array_equal(O.steady_gates(p), ka[f"{name}_init_gates"])
    assert np.array_equal(O.steady_gates(p, -55.0), ka[f"{name}_init_gates_m55"])


def test_forward_squid_ramp_bitexact():
    g = golden("fwd_squid_ramp")
    p = DF.squid_axon_params(dt=0.01)
    i = np.tile(g["i"], (int(g["T"]), 1))
    v, s, vf, gf = O.simulate(p, i, record_final=True)
    assert np.array_equal(v, g["v"]) and np.array_equal(s, g["spikes"])
    assert np.array_equal(vf, g["v_fin"]) and np.array_equal(gf, g["g_fin"])


def test_forward_config1_full_horizon_and_fp32_mode():
    g = golden("fwd_c1_one")
    p = DF.squid_axon_params(dt=0.01)
    i = np.full((10000, 1), 10.0)
    v, s = O.simulate(p, i)
    assert np.array_equal(v[:, 0], g["v"]) and np.array_equal(s[:, 0], g["spikes"])
    assert int(s.sum()) == 7
    # the reference's own float32 mode (HHParams.dtype=float32, dynamics.py:176)
    v32, s32 = O.simulate(p, i, dtype=np.float32)
    assert np.array_equal(v32[:, 0].astype(np.float32), g["v32"])
    assert np.array_equal(s32[:, 0], g["spikes32"])


@pytest.mark.parametrize("case,pname", [("fwd_rs", "rs"), ("fwd_c2", "c2")])
def test_forward_random_inputs(case, pname):
    g = golden(case)
    v, s = O.simulate(_sets()[pname], g["i"])
    assert np.array_equal(v, g["v"]) and np.array_equal(s, g["spikes"])


def test_forward_scaled_scalar_current():
    g = golden("fwd_scaled_scalar")
    p = DF.squid_axon_params(dt=0.025, rate_scale=1.7)
    v, gt = g["v0"].copy(), g["g0"].copy()
    for t in range(g["v"].shape[0]):
        v, gt, sp = O.step(p, v, gt, 14.0, step_index=t)
        assert np.array_equal(v, g["v"][t]) and np.array_equal(sp, g["spikes"][t])


def test_overflow_step_index():
    p = DF.squid_axon_params(dt=0.01)
    i = np.full((20, 2), 5.0)
    i[7, 1] = 1e308
    with pytest.raises(O.Overflow) as e:
        O.simulate(p, i * 1e10)
    assert e.value.step == 7


def _bptt_params(case):
    if case == "bptt_rs":
        return DF.cortical_rs_params(dt=0.1)
    if case == "bptt_squid_rect":
        return DF.squid_axon_params(dt=0.025, rate_scale=1.3)
    return DF.na_kdr_cal_kca_params(dt=0.02)


@pytest.mark.parametrize("case", ["bptt_rs", "bptt_squid_rect", "bptt_c2"])
def test_bptt(case):
    g = golden(case)
    p = _bptt_params(case)
    kind, width = str(g["sur"][0]) or "sigmoid-derivative", float(g["sur"][1])
    width = width if width > 0 else None
    n = g["i"].shape[1]
    v0, g0 = O.rest_state(p, n)
    full = O.bptt(p, v0, g0, g["i"], g["seed_v"], g["seed_spike"], None, kind, width)
    rel = lambda a, b: np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)
    assert rel(full["d_i"], g["d_i"]) < 1e-12
    assert rel(full["d_v0"], g["d_v0"]) < 1e-12 and rel(full["d_g0"], g["d_g0"]) < 1e-12
    assert abs(full["d_c_m"] - g["d_c_m"]) <= 1e-12 * abs(g["d_c_m"])
    assert rel(full["d_g_max"], g["d_g_max"]) < 1e-12
    assert (full["forward_calls"], full["peak_states"]) == (int(g["full_calls"]), int(g["full_peak"]))
    seg, _ = O.plan(g["i"].shape[0], int(g["budget"]))
    pl = O.bptt(p, v0, g0, g["i"], g["seed_v"], g["seed_spike"], seg, kind, width)
    assert rel(pl["d_i"], g["plan_d_i"]) < 1e-12
    assert (pl["forward_calls"], pl["peak_states"]) == (int(g["plan_calls"]), int(g["plan_peak"]))
    nos = O.bptt(p, v0, g0, g["i"], g["seed_v"], None, None, kind, width)
    assert rel(nos["d_i"], g["nos_d_i"]) < 1e-12


def test_step_backward():
    g = golden("step_backward_c2")
    p = DF.na_kdr_cal_kca_params()
    dv, dg, di, cm, gm = O.step_backward(p, g["v"], g["g"], g["i"], g["d_v"], g["d_g"],
                                         g["d_spike"], "sigmoid-derivative", O.default_width(p))
    assert np.allclose(dv, g["out_d_v"], rtol=1e-13, atol=0)
    assert np.allclose(dg, g["out_d_g"], rtol=1e-13, atol=1e-300)
    assert np.allclose(di, g["out_d_i"], rtol=1e-13, atol=0)
    assert np.isclose(cm + float(g["d_c_m_in"]), float(g["out_d_c_m"]), rtol=1e-13)
    assert np.allclose(gm + g["d_g_max_in"], g["out_d_g_max"], rtol=1e-13)


def test_readout_composition():
    g = golden("readout_rs")
    p = DF.cortical_rs_params(dt=0.1)
    drive = O.dense(g["x"], g["w"], g["b"])                 # (B, T, O)
    i_s = np.ascontiguousarray(np.moveaxis(drive, 0, 1))     # (T, B, O)
    T, B, Oo = i_s.shape
    v, s = O.simulate(p, i_s.reshape(T, -1))
    assert np.array_equal(v.reshape(T, B, Oo), g["v"])
    seed = 2.0 * v / v.size
    v0, g0 = O.rest_state(p, B * Oo)
    res = O.bptt(p, v0, g0, i_s.reshape(T, -1), seed)
    d_drive = np.moveaxis(res["d_i"].reshape(T, B, Oo), 0, 1)
    assert np.allclose(res["d_i"].reshape(T, B, Oo), g["d_i"], rtol=1e-12, atol=1e-300)
    assert np.allclose(O.dense_grad_w(d_drive, g["x"]), g["d_w"], rtol=1e-11)


def test_oracle_losses_match_reference_goldens():
    """oracle mse_loss / cross_entropy_loss (learn.py:80-107) vs the reference's outputs."""
    ka = golden("known_answers")
    loss, seed = O.mse_loss(ka["mse_pred"], ka["mse_target"])
    assert loss == float(ka["mse_loss"]) and np.array_equal(seed, ka["mse_seed"])
    loss, seed = O.cross_entropy_loss(ka["ce_logits"], ka["ce_target"])
    assert abs(loss - float(ka["ce_loss"])) <= 1e-15 * abs(loss)
    assert np.allclose(seed, ka["ce_seed"], rtol=1e-14, atol=0)


def test_oracle_morphology_matches_reference_goldens():
    """oracle morph_simulate / morph_axial (morphology.py:115-166) vs the reference."""
    from paper_2601_21407_b200 import defaults as DF
    from paper_2601_21407_b200 import morphology as M
    g = golden("morph")
    chain = M.chain_graph(5, DF.squid_axon_params(dt=0.01), 0.5)
    edges = [(chain.index(e.a), chain.index(e.b), e.g_axial) for e in chain.edges]
    params = [chain.compartments[c] for c in chain.order]
    v, s = O.morph_simulate(params, edges, g["chain_i"])
    assert np.array_equal(v, g["chain_v"]) and np.array_equal(s, g["chain_s"])
    cg = M.coincidence_graph()
    edges = [(cg.index(e.a), cg.index(e.b), e.g_axial) for e in cg.edges]
    assert np.array_equal(O.morph_axial(g["ax_v"], edges), g["ax"])
    params = [cg.compartments[c] for c in cg.order]
    for k, trial in enumerate(M.demo_trials()):
        T = int(round(40.0 / cg.dt))
        i = np.zeros((T, cg.n_compartments))
        for st in trial:
            lo, hi = int(round(st.t_on_ms / cg.dt)), int(round((st.t_on_ms + st.duration_ms) / cg.dt))
            i[lo:hi, cg.index(st.compartment)] += st.amplitude
        v, s = O.morph_simulate(params, edges, i)
        assert np.array_equal(v, g[f"demo_v{k}"]) and np.array_equal(s, g[f"demo_s{k}"])


def test_morphology_graph_validation_matches_reference():
    """CompartmentGraph checks (morphology.py:37-84) are host code: no GPU."""
    import warnings
    from paper_2601_21407_b200 import defaults as DF
    from paper_2601_21407_b200 import morphology as M
    from paper_2601_21407_b200.errors import ConfigurationError
    p = DF.squid_axon_params()
    with pytest.raises(ConfigurationError):
        M.CompartmentGraph({"a": p}, [], "zz")
    with pytest.raises(ConfigurationError):
        M.CompartmentGraph({"a": p, "b": p}, [M.Edge("a", "c", 1.0)], "a")
    with pytest.raises(ConfigurationError):
        M.CompartmentGraph({"a": p, "b": p}, [M.Edge("a", "b", -1.0)], "a")
    with pytest.raises(ConfigurationError):
        M.CompartmentGraph({"a": p, "b": p}, [], "a")           # disconnected
    with pytest.raises(ConfigurationError):
        M.CompartmentGraph({"a": p, "b": DF.squid_axon_params(dt=0.01)}, [M.Edge("a", "b", 1.0)], "a")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        M.chain_graph(3, p, 100.0)                              # dt*g/c_m > 0.5
        assert any("unstable" in str(x.message) for x in w)
    gd = M.graph_from_dict({"compartments": [{"id": "s"}, {"id": "d", "params": p.to_dict()}],
                            "edges": [{"a": "s", "b": "d", "g_axial": 1.0}], "soma": "s"})
    assert gd.order == ["s", "d"] and gd.index("d") == 1


def test_oracle_readout_model_matches_reference_goldens():
    """ReadoutModel.forward / grads (learn.py:237-274) restated with the oracle's
    dense / simulate / bptt on the reference's teacher, vs the reference."""
    g = golden("readout_fit")
    p = DF.cortical_rs_params(dt=0.1)
    x = g["filtered"]                                      # (B, T, C)
    drive = O.dense(x, g["teacher_w"], np.array([0.45]))[..., 0]
    i_s = np.ascontiguousarray(drive.T)                    # (T, B)
    v, _ = O.simulate(p, i_s)
    assert np.allclose(v.T, g["teacher_v"], rtol=1e-12, atol=1e-12)
    seed_v = np.ascontiguousarray(g["seed_pred"].T)        # scale_w = 1
    v0, g0 = O.rest_state(p, i_s.shape[1])
    res = O.bptt(p, v0, g0, i_s, seed_v)
    d_drive = res["d_i"].T
    assert np.allclose(np.einsum("bt,btc->c", d_drive, x), g["g_w"][0], rtol=1e-10)
    assert np.isclose(d_drive.sum(), g["g_b"][0], rtol=1e-10)
    assert np.isclose((g["seed_pred"] * g["teacher_v"]).sum(), g["g_sw"], rtol=1e-12)


def test_segmentation_and_split_match_reference():
    """segment_traces / split_dataset (learn.py:158-196): host logic, exact."""
    from paper_2601_21407_b200 import learn as L
    g = golden("readout_fit")
    seg = L.segment_traces(np.arange(50.0), 2.0 * np.arange(50.0), L.SegmentationScheme(7, 9))
    assert np.array_equal(np.array([a for a, _ in seg]), g["seg_in"])
    assert np.array_equal(np.array([b for _, b in seg]), g["seg_out"])
    tr, te = L.split_dataset(11, np.random.default_rng(4))
    assert np.array_equal(tr, g["split_train"]) and np.array_equal(te, g["split_test"])
    assert L.segment_traces(np.arange(5.0), np.arange(5.0), L.SegmentationScheme(7, 9)) == []
    with pytest.raises(Exception):
        L.SegmentationScheme(1, 0)
    with pytest.raises(Exception):
        L.segment_traces(np.arange(5.0), np.arange(4.0), L.SegmentationScheme(1, 1))


def test_dataset_and_history_files_roundtrip(tmp_path):
    """write/read_ndjson_dataset and write_history_csv (learn.py:384-415)."""
    from paper_2601_21407_b200 import learn as L
    rng = np.random.default_rng(0)
    x = (rng.random((3, 6, 4)) < 0.3).astype(np.float64)
    y = rng.normal(size=(3, 6))
    L.write_ndjson_dataset(tmp_path / "d.ndjson", x, y, 2)
    x2, y2, pad = L.read_ndjson_dataset(tmp_path / "d.ndjson")
    assert np.array_equal(x2, x) and np.array_equal(y2[..., 0], y) and pad == 2
    L.write_history_csv(tmp_path / "h.csv", [(0, 1.5, 0.25), (1, 0.1, 1 / 3)])
    assert (tmp_path / "h.csv").read_text() == "epoch,train_loss,val_smape\n0,1.5,0.25\n1,0.1,0.3333333333333333\n"
