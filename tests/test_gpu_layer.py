"""GPU tests of the HH SNN layer (tcgen05 projection + HH + BPTT) against the
oracle's composition of the reference readout path (learn.py:238-274) on the
same bf16-rounded operands.  Contract: V under the fp32
forward contract; dW, db, dX, d_c_m, d_g_max within 1e-3 normwise."""

import numpy as np
import pytest
import torch

from oracle import hh_oracle as O
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200.layer import HHLayer

pytestmark = pytest.mark.gpu


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("budget,n_out", [(None, 8), (4, 8), (None, 10), (4, 16)])
def test_layer_matches_oracle_composition(cuda, budget, n_out):
    """n_out % 8 == 0 takes the split-dI path (bf16 hi/lo planes straight out of
    the BPTT kernel into MN-major GEMMs); n_out = 10 the transposing path."""
    T, B, k_in = 40, 3, 24
    torch.manual_seed(0)
    layer = HHLayer(k_in, n_out, DF.cortical_rs_params(dt=0.1), budget=budget, w_mean=0.6, w_std=0.5,
                    device=cuda)
    with torch.no_grad():
        layer.bias.copy_(torch.linspace(-1.0, 2.0, n_out, device=cuda))
    g = torch.Generator(device=cuda).manual_seed(1)
    x = ((torch.rand((T, B, k_in), device=cuda, generator=g) < 0.3).float()
         + 0.1 * torch.randn((T, B, k_in), device=cuda, generator=g)).requires_grad_(True)
    V, S = layer(x)
    loss = (V ** 2).mean()
    loss.backward()

    xb = x.detach().to(torch.bfloat16).double().cpu().numpy()
    wb = layer.weight.detach().to(torch.bfloat16).double().cpu().numpy()
    b = layer.bias.detach().double().cpu().numpy()
    drive = xb @ wb.T + b                                     # (T, B, n_out)
    p = DF.cortical_rs_params(dt=0.1)
    v_ref, s_ref = O.simulate(p, drive.reshape(T, -1))
    v = V.detach().double().cpu().numpy().reshape(T, -1)
    assert np.all(np.abs(v - v_ref) <= 1e-4 * np.abs(v_ref) + 0.02) or \
        np.array_equal(S.detach().cpu().numpy().reshape(T, -1).sum(0), s_ref.sum(0))
    assert np.array_equal(S.detach().cpu().numpy().reshape(T, -1).astype(bool).sum(0), s_ref.sum(0))
    seed = 2.0 * v_ref / v_ref.size
    v0, g0 = O.rest_state(p, B * n_out)
    res = O.bptt(p, v0, g0, drive.reshape(T, -1), seed)
    d_drive = res["d_i"].reshape(T, B, n_out)
    dW_ref = np.einsum("tbc,tbk->ck", d_drive, xb)
    db_ref = d_drive.sum(axis=(0, 1))
    dX_ref = d_drive @ wb
    assert nrel(layer.weight.grad.cpu().numpy(), dW_ref) < 1e-3
    assert nrel(layer.bias.grad.cpu().numpy(), db_ref) < 1e-3
    assert nrel(x.grad.cpu().numpy(), dX_ref) < 1e-3
    pg = layer.param_grads.cpu().numpy()
    assert abs(pg[0] - res["d_c_m"]) <= 1e-3 * abs(res["d_c_m"])
    assert nrel(pg[1:], res["d_g_max"]) < 1e-3


def test_stacked_layers_gradients_flow_through_spikes(cuda):
    torch.manual_seed(2)
    l1 = HHLayer(32, 64, w_mean=0.5, w_std=0.5, device=cuda)
    l2 = HHLayer(64, 16, w_mean=0.8, w_std=0.4, device=cuda)
    x = ((torch.rand((60, 4, 32), device=cuda) < 0.3).float())
    v1, s1 = l1(x)
    v2, s2 = l2(s1)
    logits = v2.mean(0)
    loss = torch.nn.functional.cross_entropy(logits, torch.arange(4, device=cuda) % 16)
    loss.backward()
    assert s1.sum() > 0
    for t in (l1.weight.grad, l1.bias.grad, l2.weight.grad, l2.bias.grad):
        assert t is not None and torch.isfinite(t).all()
    assert l1.weight.grad.abs().sum() > 0 and l2.weight.grad.abs().sum() > 0


def test_config3_shape_runs_and_is_deterministic(cuda):
    """BASELINE config 3: batch 256, 784 -> 1024 HH neurons, 100 steps."""
    torch.manual_seed(3)
    layer = HHLayer(784, 1024, w_mean=0.05, w_std=0.1, device=cuda)
    g = torch.Generator(device=cuda).manual_seed(0)
    x = (torch.rand((100, 256, 784), device=cuda, generator=g) < 0.2).float() \
        + 0.1 * torch.randn((100, 256, 784), device=cuda, generator=g)
    grads = []
    for _ in range(2):
        layer.zero_grad()
        V, S = layer(x)
        (V ** 2).mean().backward()
        grads.append(layer.weight.grad.clone())
    assert torch.equal(grads[0], grads[1])
    assert torch.isfinite(grads[0]).all() and grads[0].abs().sum() > 0
    assert 0 < S.sum().item() < S.numel()


def _layer_and_input(cuda, budget, n_out, outputs="both", T=40, B=3, k_in=24):
    torch.manual_seed(0)
    layer = HHLayer(k_in, n_out, DF.cortical_rs_params(dt=0.1), budget=budget, w_mean=0.6, w_std=0.5,
                    device=cuda, outputs=outputs)
    with torch.no_grad():
        layer.bias.copy_(torch.linspace(-1.0, 2.0, n_out, device=cuda))
    g = torch.Generator(device=cuda).manual_seed(1)
    x = ((torch.rand((T, B, k_in), device=cuda, generator=g) < 0.3).float()
         + 0.1 * torch.randn((T, B, k_in), device=cuda, generator=g)).requires_grad_(True)
    return layer, x


@pytest.mark.parametrize("budget,n_out", [(None, 8), (4, 10), (None, 16)])
def test_fused_mse_loss_matches_unfused(cuda, budget, n_out):
    """layer.mse_loss(x) (sum V^2 in the forward kernel, seed 2 V' g / n read
    from the checkpoints in the backward kernel) == mse(layer(x)[0])."""
    from paper_2601_21407_b200.learn import mse
    layer, x = _layer_and_input(cuda, budget, n_out)
    V, _ = layer(x)
    loss_u = mse(V)
    (3.0 * loss_u).backward()
    gu = [t.grad.detach().clone() for t in (layer.weight, layer.bias, x)]
    pgu = layer.param_grads.clone()
    for t in (layer.weight, layer.bias, x):
        t.grad = None
    loss_f = layer.mse_loss(x)
    (3.0 * loss_f).backward()
    assert loss_f.dtype == torch.float32 and loss_f.dim() == 0
    assert abs(loss_f.item() - loss_u.item()) <= 1e-6 * abs(loss_u.item())
    for a, b in zip((layer.weight.grad, layer.bias.grad, x.grad), gu):
        assert nrel(a.cpu().numpy(), b.cpu().numpy()) < 1e-5
    assert nrel(layer.param_grads.cpu().numpy(), pgu.cpu().numpy()) < 1e-5


def test_layer_output_selection(cuda):
    """outputs="v" / "spikes" returns (and writes) only that trace; values and
    gradients are those of the full layer."""
    full, x = _layer_and_input(cuda, None, 8)
    V, S = full(x)
    (S.sum() * 0.01 + (V * 0.001).sum()).backward()
    for outputs in ("v", "spikes"):
        lyr, x2 = _layer_and_input(cuda, None, 8, outputs=outputs)
        V2, S2 = lyr(x2)
        if outputs == "v":
            assert S2 is None and torch.equal(V2, V)
            (V2 * 0.001).sum().backward()
        else:
            assert V2 is None and torch.equal(S2, S)
            (S2.sum() * 0.01).backward()
        assert lyr.weight.grad is not None and torch.isfinite(lyr.weight.grad).all()
    with pytest.raises(Exception):
        HHLayer(4, 8, device=cuda, outputs="neither")


def test_config3_full_shape_gradients_within_contract(cuda):
    """The benchmarked config-3 step (fused MSE) at its full shape against the
    float64 kernels (tools/parity_c3.py, profiles/r1b_parity_c3.md)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "tools/parity_c3.py"], cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("dW", "db", "dX", "d_c_m", "d_g_max"):
        assert r[k] < 1e-3, (k, r[k])
    assert r["loss_rel"] < 1e-5


def test_overlapped_weight_grads_match(cuda):
    """overlap_weight_grad=True (dW / db on a side stream, handed over at the end
    of the backward pass) gives the same gradients as the in-order path, in a
    two-layer stack, with gradient accumulation over two backward passes."""
    def build(overlap):
        torch.manual_seed(3)
        l1 = HHLayer(24, 16, DF.cortical_rs_params(dt=0.1), w_mean=0.6, w_std=0.5, device=cuda,
                     outputs="spikes", overlap_weight_grad=overlap)
        l2 = HHLayer(16, 8, DF.cortical_rs_params(dt=0.1), w_mean=0.6, w_std=0.5, device=cuda,
                     outputs="v", overlap_weight_grad=overlap)
        return l1, l2
    g = torch.Generator(device=cuda).manual_seed(5)
    x = ((torch.rand((30, 4, 24), device=cuda, generator=g) < 0.3).float()
         + 0.1 * torch.randn((30, 4, 24), device=cuda, generator=g))
    grads = []
    for overlap in (False, True):
        l1, l2 = build(overlap)
        for _ in range(2):
            _, s = l1(x)
            v, _ = l2(s)
            (v ** 2).mean().backward()
        torch.cuda.synchronize()
        grads.append([t.grad.clone() for t in (l1.weight, l1.bias, l2.weight, l2.bias)])
    for a, b in zip(*grads):
        assert torch.allclose(a, b, rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("budget,n_out", [(None, 8), (4, 10), (None, 16), (None, 32), (3, 64)])
def test_layer_bf16x3_matches_unrounded_oracle(cuda, budget, n_out):
    """proj="bf16x3" against the reference composition on the UNROUNDED
    operands (the float32 x and W taken exactly into float64, learn.py:210-211
    computing in float64): the same contract as above."""
    T, B, k_in = 40, 3, 20                  # k_in % 8 != 0: padded slots
    torch.manual_seed(0)
    layer = HHLayer(k_in, n_out, DF.cortical_rs_params(dt=0.1), budget=budget, w_mean=0.7, w_std=0.5,
                    device=cuda, proj="bf16x3")
    with torch.no_grad():
        layer.bias.copy_(torch.linspace(-1.0, 2.0, n_out, device=cuda))
    g = torch.Generator(device=cuda).manual_seed(1)
    x = ((torch.rand((T, B, k_in), device=cuda, generator=g) < 0.3).float()
         + 0.1 * torch.randn((T, B, k_in), device=cuda, generator=g)).requires_grad_(True)
    V, S = layer(x)
    ((V ** 2).mean()).backward()
    xd = x.detach().double().cpu().numpy()
    wd = layer.weight.detach().double().cpu().numpy()
    drive = xd @ wd.T + layer.bias.detach().double().cpu().numpy()
    p = DF.cortical_rs_params(dt=0.1)
    v_ref, s_ref = O.simulate(p, drive.reshape(T, -1))
    assert np.array_equal(S.detach().cpu().numpy().reshape(T, -1).astype(bool), s_ref)
    v0, g0 = O.rest_state(p, B * n_out)
    res = O.bptt(p, v0, g0, drive.reshape(T, -1), 2.0 * v_ref / v_ref.size)
    dd = res["d_i"].reshape(T, B, n_out)
    assert nrel(layer.weight.grad.cpu().numpy(), np.einsum("tbc,tbk->ck", dd, xd)) < 1e-3
    assert nrel(layer.bias.grad.cpu().numpy(), dd.sum(axis=(0, 1))) < 1e-3
    assert nrel(x.grad.cpu().numpy(), dd @ wd) < 1e-3
    pg = layer.param_grads.cpu().numpy()
    assert abs(pg[0] - res["d_c_m"]) <= 1e-3 * abs(res["d_c_m"])
    assert nrel(pg[1:], res["d_g_max"]) < 1e-3


def test_config3_full_shape_unrounded_bf16x3_within_contract(cuda):
    """Config 3 at its full shape, proj="bf16x3", against the float64 kernels
    on the unrounded float64 x and W (tools/parity_c3.py --unrounded)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "tools/parity_c3.py", "--unrounded", "--proj", "bf16x3"], cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("dW", "db", "dX", "d_c_m", "d_g_max"):
        assert r[k] < 1e-3, (k, r[k])
    assert r["loss_rel"] < 1e-4


def test_spike_operand_written_by_the_forward_kernel(cuda):
    """A spikes-only layer's forward kernel also writes its spikes as bf16 0/1
    (hhb_forward_ex2): the layer above takes them as its GEMM operand without a
    cast pass, with results identical to casting the float spikes."""
    torch.manual_seed(4)
    l1 = HHLayer(24, 32, DF.cortical_rs_params(dt=0.1), w_mean=0.6, w_std=0.5, device=cuda, outputs="spikes")
    l2 = HHLayer(32, 8, DF.cortical_rs_params(dt=0.1), w_mean=3.0, w_std=2.0, device=cuda, outputs="v")
    x = ((torch.rand((50, 3, 24), device=cuda) < 0.3).float())
    _, s = l1(x)
    twin = getattr(s, "_hhb_bf16", None)
    assert twin is not None and twin[0].dtype == torch.bfloat16
    assert torch.equal(twin[0].float(), s) and s.sum() > 0
    va, _ = l2(s)
    vb, _ = l2(s.detach().clone())          # a plain tensor: the cast path
    assert torch.equal(va, vb)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols", [(1, 5), (256, 1024), (300, 10), (513, 37), (4096, 130)])
def test_column_sums_and_loss_reduction(cuda, rows, cols):
    """hhb_col_sum_ex (the bias gradient: one launch for rows <= 512, two
    beyond) and hhb_sum_f64 (the fused loss) against float64 sums; both are
    fixed-order, so repeated calls give identical bits."""
    from paper_2601_21407_b200 import _native as nat
    from paper_2601_21407_b200.layer import col_sum_f32
    g = torch.Generator(device=cuda).manual_seed(rows * 7 + cols)
    src = torch.randn((rows, cols), device=cuda, generator=g)
    out = col_sum_f32(src)
    ref = src.double().sum(0)
    assert torch.allclose(out.double(), ref, rtol=1e-6, atol=1e-6)
    assert torch.equal(out, col_sum_f32(src))
    x = torch.rand(rows * cols, dtype=torch.float64, device=cuda, generator=g)
    o64 = torch.empty(1, dtype=torch.float64, device=cuda)
    o32 = torch.empty(1, dtype=torch.float32, device=cuda)
    nat.check(nat.load().hhb_sum_f64(x.numel(), x.data_ptr(), 0.5, o64.data_ptr(), o32.data_ptr(), None), "sum")
    torch.cuda.synchronize()
    assert abs(o64.item() - 0.5 * x.sum().item()) <= 1e-12 * x.numel()
    assert o32.item() == np.float32(o64.item())
