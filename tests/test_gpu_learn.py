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


# ---------------------------------------------------------------------------
# teacher-student readout fitting (learn.py:223-377) vs the reference's run
# ---------------------------------------------------------------------------

def _readout_task():
    from conftest import golden
    from paper_2601_21407_b200 import defaults as DF
    g = golden("readout_fit")
    neuron = DF.cortical_rs_params(dt=0.1)
    teacher = L.ReadoutModel(L.DenseLayer(g["teacher_w"], np.array([0.45])), 1.0, 0.0, neuron,
                             L.PSPKernel(tau_decay=2.0, length=64, dt=neuron.dt))
    task = L.TeacherStudentTask(teacher, g["train_inputs"], g["train_targets"], g["val_inputs"],
                                g["val_targets"], 20)
    return g, task


def test_teacher_student_task_matches_reference(cuda):
    g, _ = _readout_task()
    task = L.make_teacher_student_task(n_channels=16, n_steps=120, n_train=4, n_val=3, pad_len=20, seed=2)
    assert np.array_equal(task.train_inputs, g["train_inputs"])
    assert np.array_equal(task.val_inputs, g["val_inputs"])
    assert np.array_equal(task.teacher.dense.weights, g["teacher_w"])
    assert np.allclose(task.train_targets, g["train_targets"], rtol=1e-9, atol=1e-9)
    assert np.allclose(task.val_targets, g["val_targets"], rtol=1e-9, atol=1e-9)
    student = L.make_student(task, seed=5)
    assert np.array_equal(student.dense.weights, g["student_w0"])


@pytest.mark.parametrize("on_device", [False, True])
def test_readout_forward_and_grads_match_reference(cuda, on_device):
    g, task = _readout_task()
    t = task.teacher
    x = torch.as_tensor(g["train_inputs"], device=cuda) if on_device else g["train_inputs"]
    filt = t.filter_inputs(x)
    fh = filt.cpu().numpy() if on_device else filt
    assert np.allclose(fh, g["filtered"], rtol=1e-13, atol=1e-15)
    pred, v = t.forward(filt)
    vh = v.cpu().numpy() if on_device else v
    assert np.allclose(vh, g["teacher_v"], rtol=1e-9, atol=1e-9)
    sp = torch.as_tensor(g["seed_pred"], device=cuda) if on_device else g["seed_pred"]
    gr = t.grads(filt, sp, v)
    host = {k: (x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)) for k, x in gr.items()}
    assert host["w"].shape == (1, 16) and host["b"].shape == (1,)
    assert np.allclose(host["w"], g["g_w"], rtol=1e-8, atol=1e-12)
    assert np.allclose(host["b"], g["g_b"], rtol=1e-8)
    assert np.isclose(float(host["scale_w"]), float(g["g_sw"]), rtol=1e-9)
    assert np.isclose(float(host["scale_b"]), float(g["g_sb"]), rtol=1e-12)


def test_fit_history_and_parameters_match_reference(cuda):
    g, task = _readout_task()
    student = L.ReadoutModel(L.DenseLayer(g["student_w0"].copy(), np.zeros(1)), 1.0, 0.0, task.teacher.neuron,
                             task.teacher.kernel)
    hist = L.fit(student, task, L.TrainConfig(epochs=5, lr=2e-2))
    h = np.array(hist)
    assert np.array_equal(h[:, 0], g["history"][:, 0])
    assert np.allclose(h[:, 1:], g["history"][:, 1:], rtol=1e-7)
    assert isinstance(student.dense.weights, np.ndarray)
    assert np.allclose(student.dense.weights, g["final_w"], rtol=1e-7, atol=1e-10)
    assert np.allclose(student.dense.bias, g["final_b"], rtol=1e-7)
    assert np.isclose(student.scale_w, float(g["final_sw"]), rtol=1e-7)
    assert np.isclose(student.scale_b, float(g["final_sb"]), rtol=1e-7)
    # frozen: no parameter change, the loss repeats
    frozen = L.ReadoutModel(L.DenseLayer(g["student_w0"].copy(), np.zeros(1)), 1.0, 0.0, task.teacher.neuron,
                            task.teacher.kernel)
    hf = L.fit(frozen, task, L.TrainConfig(epochs=2, lr=2e-2, freeze=True))
    assert hf[0][1] == hf[1][1] and np.array_equal(frozen.dense.weights, g["student_w0"])
    assert np.isclose(hf[0][1], g["history"][0, 1], rtol=1e-9)


def test_readout_grad_kernel_layouts_and_empty(cuda):
    """hhb_readout_grad over both x layouts, odd channel counts, fp32, vs einsum."""
    rng = np.random.default_rng(9)
    for B, T, C in ((3, 7, 1), (5, 33, 300), (2, 1000, 64)):
        x = rng.normal(size=(B, T, C))
        dd = rng.normal(size=(T, B))
        ref_w = np.einsum("tb,btc->c", dd, x)
        for layout in ("btc", "tbc"):
            xd = torch.as_tensor(x, device=cuda)
            if layout == "tbc":
                xd = xd.permute(1, 0, 2).contiguous().permute(1, 0, 2)
            d_w = torch.empty((1, C), dtype=torch.float64, device=cuda)
            d_b = torch.empty(1, dtype=torch.float64, device=cuda)
            ws = L._readout_ws(C, cuda)
            from paper_2601_21407_b200 import _device as D, _native as nat
            ddd = torch.as_tensor(dd, device=cuda)
            nat.check(nat.load().hhb_readout_grad(nat.F64, B, T, C, xd.data_ptr(), xd.stride(0), xd.stride(1),
                                                  ddd.data_ptr(), d_w.data_ptr(), d_b.data_ptr(), ws.data_ptr(),
                                                  ws.numel() * 8, D.stream()), "grad")
            assert np.allclose(d_w.cpu().numpy()[0], ref_w, rtol=1e-11, atol=1e-11)
            assert np.isclose(d_b.item(), dd.sum(), rtol=1e-12)
            w = torch.as_tensor(rng.normal(size=C), device=cuda)
            b = torch.tensor([0.3], dtype=torch.float64, device=cuda)
            drv = L._readout_drive(xd, w, b)
            assert np.allclose(drv.cpu().numpy(), (x @ w.cpu().numpy()).T + 0.3, rtol=1e-12, atol=1e-12)


def test_fit_raises_in_reference_order(cuda):
    from paper_2601_21407_b200.errors import NumericalOverflowError, TrainingDivergedError
    g, task = _readout_task()
    bad_t = g["train_targets"].copy()
    bad_t[1, 30] = np.nan
    t2 = L.TeacherStudentTask(task.teacher, task.train_inputs, bad_t, task.val_inputs, task.val_targets, 20)
    st = L.ReadoutModel(L.DenseLayer(g["student_w0"].copy(), np.zeros(1)), 1.0, 0.0, task.teacher.neuron,
                        task.teacher.kernel)
    with pytest.raises(TrainingDivergedError) as ei:
        L.fit(st, t2, L.TrainConfig(epochs=3))
    assert ei.value.epoch == 0 and isinstance(st.dense.weights, np.ndarray)
    # a NaN before the supervised window is masked out, as in the reference
    bad_t = g["train_targets"].copy()
    bad_t[1, 3] = 1.0
    t3 = L.TeacherStudentTask(task.teacher, task.train_inputs, bad_t, task.val_inputs, task.val_targets, 20)
    h = L.fit(L.ReadoutModel(L.DenseLayer(g["student_w0"].copy(), np.zeros(1)), 1.0, 0.0, task.teacher.neuron,
                             task.teacher.kernel), t3, L.TrainConfig(epochs=1))
    assert np.isclose(h[0][1], g["history"][0, 1], rtol=1e-9)
    huge = L.ReadoutModel(L.DenseLayer(np.full((1, 16), 1e300), np.zeros(1)), 1.0, 0.0, task.teacher.neuron,
                          task.teacher.kernel)
    with pytest.raises(NumericalOverflowError):
        L.fit(huge, task, L.TrainConfig(epochs=1))


def test_fit_edge_cases(cuda):
    """epochs=0 leaves the parameters (as numpy) untouched; device inputs to
    ReadoutModel give device outputs; the cosine schedule ends at lr 0."""
    g, task = _readout_task()
    st = L.ReadoutModel(L.DenseLayer(g["student_w0"].copy(), np.zeros(1)), 1.0, 0.0, task.teacher.neuron,
                        task.teacher.kernel)
    assert L.fit(st, task, L.TrainConfig(epochs=0)) == []
    assert np.array_equal(st.dense.weights, g["student_w0"]) and st.scale_w == 1.0
    x = torch.as_tensor(g["train_inputs"], device=cuda)
    pred, v = st.forward(st.filter_inputs(x))
    assert pred.is_cuda and v.is_cuda and tuple(pred.shape) == g["train_targets"].shape
    assert L.cosine_lr(1.0, 10, 10) == pytest.approx(0.0, abs=1e-15)
    h = L.fit(st, task, L.TrainConfig(epochs=2, lr=1e-2, cosine=False))
    assert len(h) == 2 and all(np.isfinite(r[1]) and np.isfinite(r[2]) for r in h)



def test_readout_kernels_float32(cuda):
    """hhb_readout_drive / hhb_readout_grad in float32 (the kernels' second flavour)."""
    from paper_2601_21407_b200 import _device as D, _native as nat
    rng = np.random.default_rng(3)
    B, T, C = 4, 50, 37
    x = torch.as_tensor(rng.normal(size=(B, T, C)), dtype=torch.float32, device=cuda)
    w = torch.as_tensor(rng.normal(size=C), dtype=torch.float32, device=cuda)
    b = torch.tensor([0.25], dtype=torch.float32, device=cuda)
    drv = torch.empty((T, B), dtype=torch.float32, device=cuda)
    lib = nat.load()
    nat.check(lib.hhb_readout_drive(nat.F32, B, T, C, x.data_ptr(), x.stride(0), x.stride(1), w.data_ptr(),
                                    b.data_ptr(), drv.data_ptr(), D.stream()), "drive")
    ref = (x.double() @ w.double()).t() + 0.25
    assert torch.allclose(drv.double(), ref, rtol=1e-5, atol=1e-5)
    dd = torch.as_tensor(rng.normal(size=(T, B)), dtype=torch.float32, device=cuda)
    d_w = torch.empty(C, dtype=torch.float32, device=cuda)
    d_b = torch.empty(1, dtype=torch.float32, device=cuda)
    nbytes = int(lib.hhb_readout_workspace(nat.F32, C))
    ws = torch.empty(nbytes // 4, dtype=torch.float32, device=cuda)
    nat.check(lib.hhb_readout_grad(nat.F32, B, T, C, x.data_ptr(), x.stride(0), x.stride(1), dd.data_ptr(),
                                   d_w.data_ptr(), d_b.data_ptr(), ws.data_ptr(), nbytes, D.stream()), "grad")
    ref_w = torch.einsum("tb,btc->c", dd.double(), x.double())
    assert torch.allclose(d_w.double(), ref_w, rtol=1e-4, atol=1e-4)
    assert abs(d_b.item() - dd.double().sum().item()) < 1e-3
    with pytest.raises(Exception):   # workspace too small
        nat.check(lib.hhb_readout_grad(nat.F32, B, T, C, x.data_ptr(), x.stride(0), x.stride(1), dd.data_ptr(),
                                       d_w.data_ptr(), d_b.data_ptr(), ws.data_ptr(), 8, D.stream()), "grad")


def test_dense_layer_float32_runs_on_the_tcgen05_gemm(cuda):
    """learn.DenseLayer on float32 device tensors goes through hhb_gemm in the
    bf16x3 form: within 4e-5 (relative to |x||W| scale) of the float64
    x @ W.T + b of learn.py:210-211, for a batched (T, B, C) input and an
    input width that is not a multiple of 8."""
    import numpy as np
    import torch
    from paper_2601_21407_b200 import learn as L
    rng = np.random.default_rng(0)
    # (10, 4, 37): the split pass + GEMM; (64, 16, 784): >= 512 rows, x split on chip (hhb_gemm_f32a)
    # (64, 16, 784) -> 1: the readout width (output rows not 16-byte aligned: the split-pass path)
    for shape, n_out in (((10, 4, 37), 96), ((64, 16, 784), 300), ((64, 16, 784), 1)):
        layer = L.DenseLayer(rng.normal(0.05, 0.1, (n_out, shape[-1])), rng.normal(0, 1, n_out))
        x = rng.normal(0.5, 1.0, shape)
        ref = x @ layer.weights.T + layer.bias
        got = layer(torch.tensor(x, dtype=torch.float32, device=cuda))
        assert got.dtype == torch.float32 and tuple(got.shape) == shape[:-1] + (n_out,)
        xr = torch.tensor(x, dtype=torch.float32).double().numpy()        # the float32 x exactly
        wr = torch.tensor(layer.weights, dtype=torch.float32).double().numpy()
        br = torch.tensor(layer.bias, dtype=torch.float32).double().numpy()
        ref32 = xr @ wr.T + br
        scale = np.abs(xr) @ np.abs(wr).T + np.abs(br)
        assert np.max(np.abs(got.cpu().numpy() - ref32) / scale) < 4e-5    # hi/lo residuals: <= 2 x 2^-16
        assert np.allclose(got.cpu().numpy(), ref, rtol=1e-3, atol=1e-3)
    # numpy in -> numpy out, float64 (the reference's precision)
    out = layer(x)
    assert isinstance(out, np.ndarray) and np.allclose(out, ref, rtol=1e-12, atol=1e-12)
