"""GPU parity of the LIF baseline (hhb_lif_forward / hhb_lif_backward) against
the reference's golden outputs (dynamics.py:532-586, adjoint.py:197-227)."""

import numpy as np
import pytest
import torch

from conftest import golden
from paper_2601_21407_b200 import adjoint as A
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200 import dynamics as Dy

pytestmark = pytest.mark.gpu


def test_lif_simulate_matches_reference(cuda):
    g = golden("lif")
    p = DF.lif_params()
    tr = Dy.simulate(p, g["i"])
    assert np.array_equal(tr.v_series, g["v"]) and np.array_equal(tr.spike_series, g["s"])
    p32 = Dy.LIFParams(p.tau, p.v_theta, p.v_reset, p.dt, np.float32)
    tr32 = Dy.simulate(p32, g["i"].astype(np.float32))
    assert np.array_equal(tr32.v_series, g["v32"]) and np.array_equal(tr32.spike_series, g["s32"])
    # device tensors and the one-step API agree with the fused run
    td = Dy.simulate(p, torch.tensor(g["i"], device=cuda))
    assert torch.equal(td.v_series.cpu(), torch.tensor(g["v"]))
    st = Dy.init_state(p, (6,))
    for t in range(5):
        st, sp = Dy.lif_step(st, g["i"][t], p)
        assert np.array_equal(st.v, g["v"][t]) and np.array_equal(sp, g["s"][t])


def test_lif_step_backward_matches_reference(cuda):
    g = golden("lif")
    p = DF.lif_params()
    st = Dy.NeuronState(g["st_v"], np.zeros((0, 6)))
    sur = A.SurrogateSpec("sigmoid-derivative", float(g["sur_w"]))
    adj = A.AdjointState(g["d_v"], np.zeros((0, 6)), 0.0, np.zeros(0), d_spike=g["d_spike"])
    a_in, d_i = A.lif_step_backward(st, g["i"][0], p, adj, sur)
    assert np.allclose(a_in.d_v, g["bwd_dv"], rtol=1e-14, atol=0) and np.allclose(d_i, g["bwd_di"], rtol=1e-14, atol=0)
    adj2 = A.AdjointState(g["d_v"], np.zeros((0, 6)), 0.0, np.zeros(0))
    a_in2, d_i2 = A.lif_step_backward(st, g["i"][0], p, adj2, sur)
    assert np.allclose(a_in2.d_v, g["bwd2_dv"], rtol=1e-14, atol=0) and np.allclose(d_i2, g["bwd2_di"], rtol=1e-14)
