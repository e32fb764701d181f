"""GPU tests of the training plumbing (paper_2601_21407_b200.learn, SURVEY §8
f2) against the oracle restatement of learn.py:80-107."""

import numpy as np
import pytest
import torch

from oracle import hh_oracle as O
from paper_2601_21407_b200 import learn as L
from paper_2601_21407_b200.errors import UsageError

pytestmark = pytest.mark.gpu


def test_mse_loss_and_seed_match_reference(cuda):
    rng = np.random.default_rng(0)
    pred, target = rng.normal(size=(7, 5, 3)), rng.normal(size=(7, 5, 3))
    loss, seed = L.mse_loss(pred, target)
    ref_loss, ref_seed = O.mse_loss(pred, target)
    assert abs(loss - ref_loss) <= 1e-12 * abs(ref_loss)
    assert np.allclose(seed, ref_seed, rtol=1e-12, atol=0)
    with pytest.raises(UsageError):
        L.mse_loss(pred, target[:2])


def test_cross_entropy_loss_and_seed_match_reference(cuda):
    rng = np.random.default_rng(1)
    logits, y = rng.normal(size=(9, 10)) * 3, rng.integers(0, 10, size=9)
    loss, seed = L.cross_entropy_loss(logits, y)
    ref_loss, ref_seed = O.cross_entropy_loss(logits, y)
    assert abs(loss - ref_loss) <= 1e-12 * abs(ref_loss)
    assert np.allclose(seed, ref_seed, rtol=1e-10, atol=1e-15)


@pytest.mark.parametrize("with_target", [False, True])
def test_mse_autograd_gradient_is_the_reference_seed(cuda, with_target):
    g = torch.Generator(device=cuda).manual_seed(2)
    v = torch.randn((40, 3, 8), device=cuda, generator=g, dtype=torch.float64).requires_grad_(True)
    t = torch.randn((40, 3, 8), device=cuda, generator=g, dtype=torch.float64) if with_target else None
    loss = L.mse(v, t)
    loss.backward()
    ref_loss, ref_seed = O.mse_loss(v.detach().cpu().numpy(),
                                    np.zeros((40, 3, 8)) if t is None else t.cpu().numpy())
    assert abs(loss.item() - ref_loss) <= 1e-12 * ref_loss
    assert np.allclose(v.grad.cpu().numpy(), ref_seed, rtol=1e-12, atol=0)


def test_mse_autograd_fp32_fused_seed(cuda):
    """float32 path: the seed comes from hhb_scale_f32 (one pass, device scale)."""
    g = torch.Generator(device=cuda).manual_seed(4)
    v = torch.randn((100, 7, 33), device=cuda, generator=g).requires_grad_(True)   # n % 4 != 0 tail
    (3.0 * L.mse(v)).backward()
    ref = 3.0 * 2.0 * v.detach().double() / v.numel()
    assert torch.allclose(v.grad.double(), ref, rtol=1e-6, atol=0)


def test_psp_filter_smape_adam_match_reference(cuda):
    """psp_filter (lfilter order), smape and the Adam sequence with cosine lr
    against the reference's outputs (learn.py:33-151)."""
    from conftest import golden
    ka = golden("known_answers")
    y = L.psp_filter(ka["psp_in"], L.PSPKernel(2.0, 12, 0.1))
    assert np.allclose(y, ka["psp_out"], rtol=1e-14, atol=1e-16), float(np.max(np.abs(y - ka["psp_out"])))
    yd = L.psp_filter(torch.tensor(ka["psp_in"], dtype=torch.float32, device=cuda), L.PSPKernel(2.0, 12, 0.1))
    assert yd.dtype == torch.float32 and np.allclose(yd.cpu().numpy(), ka["psp_out"], rtol=1e-5, atol=1e-6)
    assert abs(L.smape(ka["smape_a"], ka["smape_b"]) - float(ka["smape"])) < 1e-12
    st = L.AdamState(lr=1e-2)
    p = {"w": ka["adam_w0"], "b": ka["adam_b0"]}
    for k in range(3):
        p = L.adam_step(p, {"w": ka["adam_gw"][k], "b": ka["adam_gb"][k]}, st, lr=L.cosine_lr(1e-2, k, 3))
    assert np.allclose(p["w"], ka["adam_w3"], rtol=1e-13, atol=1e-15)
    assert np.allclose(p["b"], ka["adam_b3"], rtol=1e-13, atol=1e-15)
