"""GPU parity of the multicompartment path (morphology.py mirror over
hhb_morph_forward) against the reference's golden traces and the oracle.
Tolerances as for single compartments: float64 V within 1e-9
relative, spikes identical; float32 under the fp32 contract."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import hh_oracle as O
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200 import morphology as M
from paper_2601_21407_b200.errors import NumericalOverflowError, UsageError
from test_gpu_forward import _close64, check_fp32_contract

pytestmark = pytest.mark.gpu


def test_fp64_chain_matches_reference(cuda):
    g = golden("morph")
    chain = M.chain_graph(5, DF.squid_axon_params(dt=0.01), 0.5)
    tr = M.simulate_morphology(chain, g["chain_i"])
    ok, err = _close64(tr.v_series, g["chain_v"])
    assert ok, err
    assert np.array_equal(tr.spike_series, g["chain_s"])


def test_fp64_coincidence_demo_matches_reference(cuda):
    """Fig. 5g-h demo: the clustered arrival fires the soma, the spread one does not."""
    g = golden("morph")
    traces = M.coincidence_experiment(M.coincidence_graph(), M.demo_trials())
    for k, tr in enumerate(traces):
        ok, err = _close64(tr.v_series, g[f"demo_v{k}"])
        assert ok, err
        assert np.array_equal(tr.spike_series, g[f"demo_s{k}"])
    assert traces[0].spike_series[:, 0].sum() == 1 and traces[1].spike_series[:, 0].sum() == 0


def test_axial_current_and_morph_step(cuda):
    g = golden("morph")
    cg = M.coincidence_graph()
    st = M.init_morph_state(cg, (4,))
    for k, s in enumerate(st.states):
        s.v[...] = g["ax_v"][k]
    ax = M.axial_current(st, cg)
    assert np.allclose(ax, g["ax"], rtol=1e-12, atol=1e-12)
    # stepping one step at a time equals the fused simulation
    rng = np.random.default_rng(3)
    i = rng.uniform(0, 20, size=(60, cg.n_compartments, 4))
    st = M.init_morph_state(cg, (4,))
    vs = []
    for t in range(60):
        st, sp = M.morph_step(st, i[t], cg, step_index=t)
        vs.append(st.potentials())
    tr = M.simulate_morphology(cg, i)
    assert np.array_equal(np.stack(vs), tr.v_series)


def test_fp32_chain_contract_and_device_tensors(cuda):
    g = golden("morph")
    p32 = DF.squid_axon_params(dt=0.01).with_(dtype=np.float32)
    chain = M.chain_graph(5, p32, 0.5)
    i = torch.tensor(g["chain_i"], dtype=torch.float32, device=cuda)
    tr = M.simulate_morphology(chain, i)
    assert tr.v_series.is_cuda
    v = tr.v_series.double().cpu().numpy().reshape(300, -1)
    s = tr.spike_series.cpu().numpy().reshape(300, -1)
    check_fp32_contract(v, s, g["chain_v"].reshape(300, -1), g["chain_s"].reshape(300, -1))


def test_large_batch_heterogeneous_tables_match_oracle(cuda):
    """A batch wider than one block (grid of 32-neuron tiles) on a graph with
    two channel tables (active soma, passive dendrites)."""
    cg = M.coincidence_graph()
    rng = np.random.default_rng(9)
    i = rng.uniform(0, 30, size=(200, cg.n_compartments, 70))
    tr = M.simulate_morphology(cg, i)
    edges = [(cg.index(e.a), cg.index(e.b), e.g_axial) for e in cg.edges]
    v_ref, s_ref = O.morph_simulate([cg.compartments[c] for c in cg.order], edges, i)
    ok, err = _close64(tr.v_series, v_ref)
    assert ok, err
    assert np.array_equal(tr.spike_series, s_ref)


def test_morphology_errors(cuda):
    cg = M.coincidence_graph()
    with pytest.raises(UsageError):
        M.simulate_morphology(cg, np.zeros((10, 3)))
    with pytest.raises(NumericalOverflowError):
        M.simulate_morphology(cg, np.full((50, cg.n_compartments), 1e300))
