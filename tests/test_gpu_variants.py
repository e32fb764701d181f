"""Kernel variants kept behind environment knobs (DESIGN.md §3, §8 "tried"):
each must stay correct even though the default build does not run it.

* HHB_JIT_POLY_EXP=k — k shared rate exponentials of the merged forward on the
  FMA pipe (degree-6 polynomial): the float32 contract against the reference.
* HHB_JIT_BWD_PAIR=1 — the paired (f32x2) adjoint step: gradients equal the
  default (scalar) kernel's within float32 rounding.
* HHB_LAYER_CHUNKS=c — the time-chunked projection / forward pipeline of
  HHLayer: identical gradients to the unchunked step.
* HHB_PDL=1 — programmatic dependent launch of the layer chain: bit-identical
  results (a launch-order change only; run in a subprocess, the switch is read
  once per process).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import golden, requires_jit
from paper_2601_21407_b200 import adjoint as A
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200 import dynamics as Dy

pytestmark = [pytest.mark.gpu, requires_jit]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture
def env(monkeypatch):
    return monkeypatch


@pytest.mark.parametrize("k", [1, 3])
def test_polynomial_exp2_forward_meets_the_contract(cuda, env, k):
    from test_gpu_forward import check_fp32_contract
    env.setenv("HHB_JIT_POLY_EXP", str(k))
    g = golden("fwd_c2")
    i = g["i"] if g["i"].ndim == 2 else np.tile(g["i"], (int(g["T"]), 1))
    tr = Dy.simulate(DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32), i)
    check_fp32_contract(tr.v_series, tr.spike_series, g["v"], g["spikes"])


def test_paired_adjoint_step_matches_scalar(cuda, env):
    p = DF.cortical_rs_params(dt=0.1).with_(dtype=np.float32)
    n, T = 4096, 60
    g = torch.Generator(device=cuda).manual_seed(3)
    i = 7.8 + 3.0 * torch.randn((T, n), device=cuda, generator=g)
    sv = 1e-3 * torch.randn((T, n), device=cuda, generator=g)
    s0 = Dy.init_state(p, (n,))
    s0 = Dy.NeuronState(torch.as_tensor(s0.v, dtype=torch.float32, device=cuda),
                        torch.as_tensor(s0.gates, dtype=torch.float32, device=cuda))
    ref = A.backward_through_time(p, s0, i, sv)
    env.setenv("HHB_JIT_BWD_PAIR", "1")
    got = A.backward_through_time(p, s0, i, sv)
    assert torch.allclose(got.d_i, ref.d_i, rtol=1e-4, atol=1e-9)
    for a, b in zip(np.atleast_1d(got.d_g_max), np.atleast_1d(ref.d_g_max)):
        assert abs(a - b) <= 1e-4 * abs(b) + 1e-12
    assert abs(got.d_c_m - ref.d_c_m) <= 1e-4 * abs(ref.d_c_m) + 1e-12


def _layer_grads(cuda, chunks, env, proj="bf16"):
    from paper_2601_21407_b200.layer import HHLayer
    env.setenv("HHB_LAYER_CHUNKS", str(chunks))
    torch.manual_seed(0)
    layer = HHLayer(784, 1024, w_mean=0.05, w_std=0.1, device=cuda, proj=proj)
    g = torch.Generator(device=cuda).manual_seed(0)
    x = ((torch.rand((100, 256, 784), device=cuda, generator=g) < 0.2).float()
         + 0.1 * torch.randn((100, 256, 784), device=cuda, generator=g))
    loss = layer.mse_loss(x)
    loss.backward()
    torch.cuda.synchronize()
    return float(loss.detach()), layer.weight.grad.clone(), layer.bias.grad.clone()


@pytest.mark.parametrize("proj", ["bf16", "bf16x3"])
def test_time_chunked_layer_pipeline_matches(cuda, env, proj):
    # bf16x3: the on-chip split GEMM (hhb_gemm_f32a) on row chunks of x
    l1, w1, b1 = _layer_grads(cuda, 1, env, proj)
    l4, w4, b4 = _layer_grads(cuda, 4, env, proj)
    # the forward states are the same launches' states, chunk by chunk: the
    # gradients are identical; the loss's fp64 partial sums regroup per chunk
    assert torch.equal(w1, w4) and torch.equal(b1, b4)
    assert abs(l1 - l4) <= 1e-12 * abs(l1)


_PDL_CHILD = r"""
import json, sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2601_21407_b200.layer import HHLayer
dev = torch.device("cuda", 0)
torch.manual_seed(0)
layer = HHLayer(784, 512, w_mean=0.05, w_std=0.1, device=dev, proj=sys.argv[2])
g = torch.Generator(device=dev).manual_seed(0)
x = ((torch.rand((50, 128, 784), device=dev, generator=g) < 0.2).float()
     + 0.1 * torch.randn((50, 128, 784), device=dev, generator=g))
loss = layer.mse_loss(x)
loss.backward()
print(json.dumps({"loss": float(loss), "w": float(layer.weight.grad.double().abs().sum()),
                  "w0": layer.weight.grad[:4, :4].flatten().tolist(), "b": layer.bias.grad[:8].tolist()}))
"""


@pytest.mark.parametrize("proj", ["bf16", "bf16x3"])
def test_programmatic_dependent_launch_is_bit_identical(cuda, proj):
    out = {}
    for pdl in ("0", "1"):
        e = dict(os.environ, HHB_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", _PDL_CHILD, ROOT, proj], env=e, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[pdl] = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["0"] == out["1"]


@pytest.mark.parametrize("n_out", [12, 10])
def test_onchip_split_projection_matches_split_pass(cuda, env, n_out):
    """bf16x3 layer with >= 512 rows: the on-chip split GEMM (n_out a multiple
    of 4) against HHB_LAYER_FUSED_SPLIT=0 (the split pass + K = 3k GEMM): the
    same three products, accumulated in another order -- gradients agree to
    float32 rounding; n_out = 10 (unaligned output rows) takes the split pass."""
    from paper_2601_21407_b200.layer import HHLayer

    def run():
        torch.manual_seed(0)
        layer = HHLayer(64, n_out, w_mean=0.3, w_std=0.2, device=cuda, proj="bf16x3")
        g = torch.Generator(device=cuda).manual_seed(1)
        x = ((torch.rand((40, 16, 64), device=cuda, generator=g) < 0.3).float()
             + 0.1 * torch.randn((40, 16, 64), device=cuda, generator=g))
        layer.mse_loss(x).backward()
        torch.cuda.synchronize()
        return layer.weight.grad.double(), layer.bias.grad.double()

    w1, b1 = run()
    env.setenv("HHB_LAYER_FUSED_SPLIT", "0")
    w0, b0 = run()
    assert torch.allclose(w1, w0, rtol=1e-4, atol=1e-6 * float(w0.abs().max()))
    assert torch.allclose(b1, b0, rtol=1e-4, atol=1e-6 * float(b0.abs().max()))
