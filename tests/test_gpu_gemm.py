"""GPU tests of the tcgen05 projection GEMM (hhb_gemm) against fp64 references
on the same (bf16- / tf32-rounded) operands: D = A B^T + bias."""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2601_21407_b200 import _native as nat

pytestmark = pytest.mark.gpu


def gemm(A, B, bias=None, splits=1, kind=0):
    M, K = A.shape
    N = B.shape[0]
    D = torch.empty((M, N), dtype=torch.float32, device=A.device)
    lib = nat.load()
    ws_n = int(lib.hhb_gemm_workspace(M, N, splits))
    ws = torch.empty(max(1, ws_n), dtype=torch.float32, device=A.device)
    rc = lib.hhb_gemm(kind, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                      None if bias is None else bias.data_ptr(), D.data_ptr(), N, splits, ws.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
    nat.check(rc, "hhb_gemm")
    return D


def tf32_round(x):
    """Round-to-nearest tf32 (10-bit mantissa) of an fp32 tensor, as float64."""
    b = x.contiguous().view(torch.int32).to(torch.int64)
    b = (b + 0x1000) & ~0x1FFF
    return b.to(torch.int32).view(torch.float32).double()


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (1000, 200, 104), (25600, 1024, 784), (257, 10, 2048),
                                   (300, 2048, 2048)])
def test_bf16_gemm_matches_reference(cuda, M, N, K):
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N)
    A = torch.randn((M, K), device=cuda, generator=g).to(torch.bfloat16)
    B = torch.randn((N, K), device=cuda, generator=g).to(torch.bfloat16)
    bias = torch.randn(N, device=cuda, generator=g)
    D = gemm(A, B, bias)
    ref = A.double() @ B.double().T + bias.double()
    err = (D.double() - ref).norm() / ref.norm()
    # bf16 products are exact in fp32; the tensor cores' fp32 accumulation
    # error grows ~linearly with K (measured 2e-7 at K=256, 2e-6 at K=2048,
    # 9e-6 at K=8192: tools/gemm_err.py)
    assert err < 2e-6 * max(1.0, K / 1024), float(err)
    assert torch.isfinite(D).all()


def test_bf16_gemm_without_bias_and_tail_rows(cuda):
    A = torch.randn((77, 96), device=cuda).to(torch.bfloat16)
    B = torch.randn((33, 96), device=cuda).to(torch.bfloat16)
    D = gemm(A, B)
    ref = A.double() @ B.double().T
    assert ((D.double() - ref).abs().max() / ref.abs().max()) < 1e-6


@pytest.mark.parametrize("M,N,K,splits", [(1024, 784, 25600, 8), (10, 2048, 25600, 16), (256, 256, 512, 1)])
def test_tf32_split_k_gemm_is_deterministic(cuda, M, N, K, splits):
    g = torch.Generator(device=cuda).manual_seed(3)
    A = torch.randn((M, K), device=cuda, generator=g)
    B = torch.randn((N, K), device=cuda, generator=g)
    D1 = gemm(A, B, splits=splits, kind=1)
    D2 = gemm(A, B, splits=splits, kind=1)
    assert torch.equal(D1, D2)
    ref_x = A.double() @ B.double().T
    err_x = float((D1.double() - ref_x).norm() / ref_x.norm())
    # tf32 operands (10-bit mantissa): measured ~8e-4 normwise vs exact fp64
    assert err_x < 2e-3, err_x
    Ds = gemm(A, B, splits=1, kind=1)
    assert float((Ds - D1).norm() / D1.norm()) < 2e-4


def test_transpose_cast_colsum(cuda):
    lib = nat.load()
    x = torch.randn((333, 129), device=cuda)
    t = torch.empty((129, 333), device=cuda)
    nat.check(lib.hhb_transpose(0, 333, 129, x.data_ptr(), 129, t.data_ptr(), 333, None), "t")
    torch.cuda.synchronize()
    assert torch.equal(t, x.T.contiguous())
    tb = torch.empty((129, 333), dtype=torch.bfloat16, device=cuda)
    nat.check(lib.hhb_transpose(1, 333, 129, x.data_ptr(), 129, tb.data_ptr(), 333, None), "t")
    torch.cuda.synchronize()
    assert torch.equal(tb, x.T.contiguous().to(torch.bfloat16))
    cb = torch.empty_like(x, dtype=torch.bfloat16)
    nat.check(lib.hhb_cast_bf16(x.numel(), x.data_ptr(), cb.data_ptr(), None), "c")
    torch.cuda.synchronize()
    assert torch.equal(cb, x.to(torch.bfloat16))
    s = torch.zeros(129, dtype=torch.float64, device=cuda)
    scratch = torch.empty(int(lib.hhb_col_sum_scratch(333, 129)), dtype=torch.float64, device=cuda)
    nat.check(lib.hhb_col_sum(333, 129, x.data_ptr(), 129, s.data_ptr(), scratch.data_ptr(), None), "s")
    torch.cuda.synchronize()
    assert torch.allclose(s, x.double().sum(0), rtol=1e-12, atol=1e-9)


def gemm_ex(A, B, *, a_mn=False, b_mn=False, A2=None, bias=None, splits=1):
    """D = (A (+A2)) B^T; A given as (M, K) (K-major) or (K, M) (a_mn), B as (N, K) or (K, N)."""
    M = A.shape[1] if a_mn else A.shape[0]
    K = A.shape[0] if a_mn else A.shape[1]
    N = B.shape[1] if b_mn else B.shape[0]
    D = torch.empty((M, N), dtype=torch.float32, device=A.device)
    lib = nat.load()
    ws_n = int(lib.hhb_gemm_workspace(M, N, splits))
    ws = torch.empty(max(1, ws_n), dtype=torch.float32, device=A.device)
    flags = (1 if a_mn else 0) | (2 if b_mn else 0)
    rc = lib.hhb_gemm_ex(flags, M, N, K, A.data_ptr(), None if A2 is None else A2.data_ptr(), A.stride(0),
                         B.data_ptr(), B.stride(0), None if bias is None else bias.data_ptr(), D.data_ptr(), N,
                         splits, ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    nat.check(rc, "hhb_gemm_ex")
    return D


@pytest.mark.parametrize("a_mn,b_mn,dual", [(a, b, d) for a in (False, True) for b in (False, True)
                                            for d in (False, True)])
@pytest.mark.parametrize("M,N,K,splits", [(1024, 784, 2560, 4), (300, 200, 136, 1), (128, 64, 64, 1)])
def test_gemm_ex_layouts_and_dual_operand(cuda, a_mn, b_mn, dual, M, N, K, splits):
    """MN-major operands (UMMA descriptors with LBO = 8 KB chunks) and the
    dual-A accumulation against an fp64 product of the same bf16 values."""
    g = torch.Generator(device=cuda).manual_seed(M + N + K + 2 * a_mn + b_mn)
    Am = torch.randn((M, K), device=cuda, generator=g)
    hi = Am.to(torch.bfloat16)
    lo = (Am - hi.float()).to(torch.bfloat16)
    Bm = torch.randn((N, K), device=cuda, generator=g).to(torch.bfloat16)
    bias = torch.randn(N, device=cuda, generator=g)
    def mn(x):   # (R, K) -> (K, R) view with a 16-byte aligned row pitch
        r = x.shape[0]
        buf = torch.zeros((x.shape[1], (r + 7) // 8 * 8), dtype=x.dtype, device=x.device)
        buf[:, :r] = x.T
        return buf[:, :r]

    def km(x):
        k = x.shape[1]
        buf = torch.zeros((x.shape[0], (k + 7) // 8 * 8), dtype=x.dtype, device=x.device)
        buf[:, :k] = x
        return buf[:, :k]

    A1 = mn(hi) if a_mn else km(hi)
    A2 = (mn(lo) if a_mn else km(lo)) if dual else None
    B1 = mn(Bm) if b_mn else km(Bm)
    D = gemm_ex(A1, B1, a_mn=a_mn, b_mn=b_mn, A2=A2, bias=bias, splits=splits)
    Aref = hi.double() + (lo.double() if dual else 0.0)
    ref = Aref @ Bm.double().T + bias.double()
    err = float((D.double() - ref).norm() / ref.norm())
    assert err < 2e-6 * max(1.0, K / 1024), err
    if dual:   # the pair carries ~16 mantissa bits of the fp32 operand
        full = Am.double() @ Bm.double().T + bias.double()
        assert float((D.double() - full).norm() / full.norm()) < 5e-5


@pytest.mark.parametrize("rows,cols", [(300, 784), (33, 20), (64, 24)])
def test_split3_slots(cuda, rows, cols):
    """hhb_split3_bf16 (vectorised when cols % 8 == 0, scalar otherwise):
    slots [hi | lo | hi] (order 0) and [hi | hi | lo] (order 1), hi = bf16(x),
    lo = bf16(x - hi), pad columns untouched (zero)."""
    from paper_2601_21407_b200.layer import split3_padded
    x = torch.randn((rows, cols), device=cuda) * 3.0
    hi = x.to(torch.bfloat16)
    lo = (x - hi.float()).to(torch.bfloat16)
    for order in (0, 1):
        out, kp = split3_padded(x, order)
        assert out.shape == (rows, 3 * kp) and kp % 8 == 0 and kp >= cols
        s0, s1, s2 = out[:, :cols], out[:, kp:kp + cols], out[:, 2 * kp:2 * kp + cols]
        assert torch.equal(s0, hi)
        assert torch.equal(s1, lo if order == 0 else hi)
        assert torch.equal(s2, hi if order == 0 else lo)
        if kp > cols:
            assert not out[:, cols:kp].float().any()


@pytest.mark.parametrize("M,N,P", [(1024, 784, 1024), (512, 96, 32), (256, 40, 64)])
def test_gemm_k_switch_concatenates_a(cuda, M, N, P):
    """hhb_gemm_ex2: K-major A for k < k_switch, A2 (same pitch) at k - k_switch
    above -- here the layer's dX: A rows [hi | lo] (2P), then hi again, against
    MN-major B rows [B0; B1; B2] (3P x N); equal to the explicit concatenation."""
    from paper_2601_21407_b200.layer import B_MN, gemm_ex, gemm_ex2
    torch.manual_seed(1)
    H = torch.randn((M, 2 * P), device=cuda).to(torch.bfloat16)
    Bm = torch.randn((3 * P, N), device=cuda).to(torch.bfloat16).contiguous()
    got = gemm_ex2(B_MN, M, N, 3 * P, H, H, 2 * P, Bm, N, 2 * P)
    a_cat = torch.cat([H, H[:, :P]], dim=1).float()
    ref = a_cat @ Bm.float()
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-3), float((got - ref).abs().max())
    # the explicit concatenation through the plain GEMM agrees bit for bit
    explicit = gemm_ex(B_MN, M, N, 3 * P, torch.cat([H, H[:, :P]], dim=1).contiguous(), None, 3 * P, Bm, N)
    assert torch.equal(got, explicit)



def test_split3_stacked_rows(cuda):
    """order 2: three row blocks [hi; hi; lo] of `slot` rows (the dX B operand)."""
    from paper_2601_21407_b200 import _native as nat
    for rows, cols, P, ld in ((10, 20, 16, 24), (64, 784, 64, 784)):
        x = torch.randn((rows, cols), device=cuda)
        out = torch.zeros((3 * P, ld), dtype=torch.bfloat16, device=cuda)
        nat.check(nat.load().hhb_split3_bf16(rows, cols, x.data_ptr(), cols, out.data_ptr(), ld, P, 2,
                                             torch.cuda.current_stream().cuda_stream), "split3")
        hi = x.to(torch.bfloat16)
        lo = (x - hi.float()).to(torch.bfloat16)
        assert torch.equal(out[:rows, :cols], hi) and torch.equal(out[P:P + rows, :cols], hi)
        assert torch.equal(out[2 * P:2 * P + rows, :cols], lo)
        assert not out[rows:P].float().any() and not out[:, cols:].float().any()


@pytest.mark.parametrize("M,N,K,bias,splits", [(512, 256, 784, False, 0), (1000, 300, 96, True, 0),
                                               (25600, 1024, 784, True, 0), (4096, 784, 784, False, 0),
                                               (512, 256, 8192, False, 4), (2048, 2048, 2048, True, 0)])
def test_fp32_a_gemm_converts_on_chip(cuda, M, N, K, bias, splits):
    """hhb_gemm_f32a / HHB_GEMM_A_F32: fp32 x rounded to bf16 inside the GEMM
    gives the cast-then-GEMM result bit for bit; with B_lo it is the fp32-class
    three-product form (hi.W_hi + lo.W_hi + hi.W_lo) within the error of the
    unfused one against float64, and the hi / lo operand it writes out equals
    the split pass's (hhb_split3_bf16) slots."""
    from paper_2601_21407_b200.layer import _stream, _workspace, gemm, split3_padded, to_bf16_padded
    lib = nat.load()
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    x = torch.randn((M, K), device=cuda, generator=g)
    w = torch.randn((N, K), device=cuda, generator=g) * 0.05
    b = torch.randn(N, device=cuda, generator=g) if bias else None
    ws = _workspace(int(lib.hhb_gemm_workspace(M, N, max(splits, 32))), cuda)
    wb = to_bf16_padded(w)

    def f32a(B, Blo, ldb, xs=None, xs_ld=0, slot=0):
        out = torch.empty((M, N), device=cuda)
        nat.check(lib.hhb_gemm_f32a(M, N, K, x.data_ptr(), K, B.data_ptr(), None if Blo is None else Blo.data_ptr(),
                                    ldb, None if b is None else b.data_ptr(), out.data_ptr(), N, splits,
                                    ws.data_ptr(), None if xs is None else xs.data_ptr(), xs_ld, slot, _stream()),
                  "f32a")
        return out

    ref = gemm(to_bf16_padded(x), wb, K, bias=b, splits=splits if splits > 0 else None)
    assert torch.equal(f32a(wb, None, wb.stride(0)), ref)
    w3, kp = split3_padded(w, 1)                      # [W_hi | W_hi | W_lo]
    xs = torch.zeros((M, 2 * kp), dtype=torch.bfloat16, device=cuda)
    got3 = f32a(w3, w3[:, 2 * kp:], w3.stride(0), xs, xs.stride(0), kp)
    xb3, _ = split3_padded(x, 0)                      # [x_hi | x_lo | x_hi]
    ref3 = gemm(xb3, w3, 3 * kp, bias=b)
    exact = x.double() @ w.double().T + (b.double() if b is not None else 0)
    scale = exact.abs().max()
    assert (got3.double() - exact).abs().max() / scale < 4 * (ref3.double() - exact).abs().max() / scale + 1e-6
    assert torch.equal(xs[:, :K], xb3[:, :K]) and torch.equal(xs[:, kp:kp + K], xb3[:, kp:kp + K])


@pytest.mark.parametrize("R,n_out,k_in,splits", [(1024, 512, 384, 0), (4096, 600, 200, 0), (25600, 1024, 784, 0),
                                                 (2048, 512, 784, 3)])
def test_fp32_b_weight_gradient_gemm_bf16(cuda, R, n_out, k_in, splits):
    """hhb_gemm_f32b with split_b = 0 (proj="bf16"): (dI_hi + dI_lo)^T bf16(x)
    equals the dual GEMM over the cast x bit for bit (the same products, in
    the same k order)."""
    from paper_2601_21407_b200.layer import A_MN, B_MN, _stream, _workspace, gemm_ex, to_bf16_padded
    lib = nat.load()
    g = torch.Generator(device=cuda).manual_seed(R + n_out + 1)
    dI = torch.randn((R, n_out), device=cuda, generator=g) * 1e-3
    x = torch.randn((R, k_in), device=cuda, generator=g)
    hi = dI.to(torch.bfloat16)
    lo = (dI - hi.float()).to(torch.bfloat16)
    xb = to_bf16_padded(x)
    ws = _workspace(int(lib.hhb_gemm_workspace(n_out, k_in, max(splits, 32))), cuda)
    ref = gemm_ex(A_MN | B_MN, n_out, k_in, R, hi, lo, n_out, xb, xb.stride(0), splits=splits if splits else None)
    out = torch.empty((n_out, k_in), device=cuda)
    nat.check(lib.hhb_gemm_f32b(n_out, k_in, R, hi.data_ptr(), lo.data_ptr(), n_out, x.data_ptr(), k_in, 0,
                                out.data_ptr(), k_in, splits, ws.data_ptr(), _stream()), "f32b")
    torch.cuda.synchronize()
    exact = dI.double().T @ x.double()
    scale = exact.abs().max()
    assert (out.double() - exact).abs().max() / scale <= 1.01 * (ref.double() - exact).abs().max() / scale + 1e-7


@pytest.mark.parametrize("R,n_out,k_in,splits", [(1024, 512, 384, 0), (4096, 600, 200, 0), (25600, 1024, 784, 0),
                                                 (2048, 512, 784, 3), (1000, 520, 136, 0)])
def test_fp32_b_weight_gradient_gemm(cuda, R, n_out, k_in, splits):
    """hhb_gemm_f32b: dW = (dI_hi + dI_lo)^T x_hi + dI_hi^T x_lo with the fp32 x
    split on chip (MN-major) -- within the error of the two-GEMM composition
    over the split pass's x_hi / x_lo against float64."""
    from paper_2601_21407_b200.layer import A_MN, B_MN, _stream, _workspace, gemm_ex, split3_padded
    lib = nat.load()
    g = torch.Generator(device=cuda).manual_seed(R + n_out)
    dI = torch.randn((R, n_out), device=cuda, generator=g) * 1e-3
    x = torch.randn((R, k_in), device=cuda, generator=g)
    hi = dI.to(torch.bfloat16)
    lo = (dI - hi.float()).to(torch.bfloat16)
    xs3, kp = split3_padded(x, 0)
    ref = gemm_ex(A_MN | B_MN, n_out, k_in, R, hi, lo, n_out, xs3, xs3.stride(0))
    ref += gemm_ex(A_MN | B_MN, n_out, k_in, R, hi, None, n_out, xs3[:, kp:], xs3.stride(0))
    out = torch.empty((n_out, k_in), device=cuda)
    ws = _workspace(int(lib.hhb_gemm_workspace(n_out, k_in, max(splits, 32))), cuda)
    nat.check(lib.hhb_gemm_f32b(n_out, k_in, R, hi.data_ptr(), lo.data_ptr(), n_out, x.data_ptr(), k_in, 1,
                                out.data_ptr(), k_in, splits, ws.data_ptr(), _stream()), "f32b")
    exact = dI.double().T @ x.double()
    scale = exact.abs().max()
    assert (out.double() - exact).abs().max() / scale < 4 * (ref.double() - exact).abs().max() / scale + 1e-6
