"""Fused fp32-A GEMM (HHB_GEMM_A_F32[_SPLIT]) against the unfused paths: bit
identity for the bf16 cast form, the three-product form against float64, and
timing of both at the config-3 projection shape."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_21407_b200 import _native as nat
from paper_2601_21407_b200.layer import _workspace, gemm, to_bf16_padded, split3_padded, _stream

A_F32, A_SPLIT = 4, 8
dev = torch.device("cuda", 0)
lib = nat.load()


def fused(x, wb, bias=None, wlo=None, splits=0):
    M, K = x.shape
    N = wb.shape[0]
    out = torch.empty((M, N), dtype=torch.float32, device=dev)
    ws_n = int(lib.hhb_gemm_workspace(M, N, splits if splits > 0 else 32))
    ws = _workspace(ws_n, dev) if ws_n else None
    flags = A_F32 | (A_SPLIT if wlo is not None else 0)
    nat.check(lib.hhb_gemm_ex(flags, M, N, K, x.data_ptr(), None if wlo is None else wlo.data_ptr(), x.stride(0),
                              wb.data_ptr(), wb.stride(0), None if bias is None else bias.data_ptr(), out.data_ptr(),
                              N, splits, None if ws is None else ws.data_ptr(), _stream()), "fused")
    return out


def check(M, N, K, with_bias, splits=0):
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    x = torch.randn((M, K), device=dev, generator=g)
    w = torch.randn((N, K), device=dev, generator=g) * 0.05
    b = torch.randn(N, device=dev, generator=g) if with_bias else None
    wb = to_bf16_padded(w)
    ref = gemm(to_bf16_padded(x), wb, K, bias=b, splits=splits if splits > 0 else None)
    got = fused(x, wb, b, splits=splits)
    torch.cuda.synchronize()
    same = torch.equal(ref, got)
    # three-product form vs float64 and vs the unfused slots GEMM
    whi = to_bf16_padded(w)
    wlo = to_bf16_padded((w - w.to(torch.bfloat16).float()).contiguous())
    got3 = fused(x, whi, b, wlo=wlo, splits=splits)
    xb3, kp = split3_padded(x, 0)
    wb3, _ = split3_padded(w, 1)
    ref3 = gemm(xb3, wb3, 3 * kp, bias=b)
    exact = x.double() @ w.double().T + (b.double() if b is not None else 0)
    torch.cuda.synchronize()
    e3 = ((got3.double() - exact).abs().max() / exact.abs().max()).item()
    r3 = ((ref3.double() - exact).abs().max() / exact.abs().max()).item()
    print(f"M={M} N={N} K={K} bias={with_bias} splits={splits}: bf16 bit-identical={same}; "
          f"3-product rel err {e3:.2e} (unfused {r3:.2e})", flush=True)
    return same and e3 < 4 * r3 + 1e-6


def check_xs(M, N, K):
    """the converted operand written out = the split pass's slots 0 / 1"""
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn((M, K), device=dev, generator=g)
    w = torch.randn((N, K), device=dev, generator=g) * 0.05
    wb3, kp = split3_padded(w, 1)
    xs = torch.zeros((M, 2 * kp), dtype=torch.bfloat16, device=dev)
    out = torch.empty((M, N), device=dev)
    ws = _workspace(int(lib.hhb_gemm_workspace(M, N, 32)), dev)
    nat.check(lib.hhb_gemm_f32a(M, N, K, x.data_ptr(), K, wb3.data_ptr(), wb3[:, 2 * kp:].data_ptr(), wb3.stride(0),
                                None, out.data_ptr(), N, 0, ws.data_ptr(), xs.data_ptr(), xs.stride(0), kp,
                                _stream()), "f32a")
    ref, _ = split3_padded(x, 0)
    torch.cuda.synchronize()
    same = torch.equal(xs[:, :K], ref[:, :K]) and torch.equal(xs[:, kp:kp + K], ref[:, kp:kp + K])
    print(f"xs M={M} N={N} K={K}: hi/lo written = split pass: {same}", flush=True)
    return same


ok = True
for case in [(512, 256, 784), (25600, 1024, 784), (1000, 300, 96)]:
    ok = check_xs(*case) and ok
for case in [(512, 256, 784, False), (512, 256, 784, True), (1000, 300, 100, True), (25600, 1024, 784, True),
             (4096, 784, 784, False), (512, 256, 8192, False, 4), (2048, 2048, 2048, True)]:
    ok = check(*case) and ok


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


M, N, K = 25600, 1024, 784
x = torch.randn((M, K), device=dev)
w = torch.randn((N, K), device=dev) * 0.05
b = torch.zeros(N, device=dev)
wb = to_bf16_padded(w)
whi = w.to(torch.bfloat16).contiguous()
wlo = (w - whi.float()).to(torch.bfloat16).contiguous()
print("config-3 projection, us per call:")
print(" cast + bf16 GEMM   %.1f" % timeit(lambda: gemm(to_bf16_padded(x), wb, K, bias=b)))
print(" fused bf16         %.1f" % timeit(lambda: fused(x, wb, b)))
print(" split3 + GEMM(3K)  %.1f" % timeit(lambda: gemm(split3_padded(x, 0)[0], split3_padded(w, 1)[0], 3 * K, bias=b)))
print(" fused 3-product    %.1f" % timeit(lambda: fused(x, whi, b, wlo=wlo)))
kp3 = K
xs3 = torch.empty((M, 2 * kp3), dtype=torch.bfloat16, device=dev)
out3 = torch.empty((M, N), device=dev)


def fused_xs():
    nat.check(lib.hhb_gemm_f32a(M, N, K, x.data_ptr(), K, whi.data_ptr(), wlo.data_ptr(), whi.stride(0), b.data_ptr(),
                                out3.data_ptr(), N, 0, None, xs3.data_ptr(), xs3.stride(0), kp3, _stream()), "xs")


print(" fused 3-product + x_hi/x_lo written  %.1f" % timeit(fused_xs))

# weight-gradient form (hhb_gemm_f32b): dW = (dI_hi + dI_lo)^T x_hi + dI_hi^T x_lo with x fp32
from paper_2601_21407_b200.layer import gemm_ex, A_MN, B_MN


def check_f32b(R, n_out, k_in, splits=0):
    g = torch.Generator(device=dev).manual_seed(R + n_out)
    dI = torch.randn((R, n_out), device=dev, generator=g) * 1e-3
    xf = torch.randn((R, k_in), device=dev, generator=g)
    hi = dI.to(torch.bfloat16)
    lo = (dI - hi.float()).to(torch.bfloat16)
    xs3, kp = split3_padded(xf, 0)
    ref = gemm_ex(A_MN | B_MN, n_out, k_in, R, hi, lo, n_out, xs3, xs3.stride(0))
    ref += gemm_ex(A_MN | B_MN, n_out, k_in, R, hi, None, n_out, xs3[:, kp:], xs3.stride(0))
    out = torch.empty((n_out, k_in), device=dev)
    ws = _workspace(int(lib.hhb_gemm_workspace(n_out, k_in, 32)), dev)
    fn = lambda: nat.check(lib.hhb_gemm_f32b(n_out, k_in, R, hi.data_ptr(), lo.data_ptr(), n_out, xf.data_ptr(),
                                             k_in, 1, out.data_ptr(), k_in, splits, ws.data_ptr(), _stream()), "f32b")
    fn()
    exact = dI.double().T @ xf.double()
    torch.cuda.synchronize()
    e = ((out.double() - exact).abs().max() / exact.abs().max()).item()
    r = ((ref.double() - exact).abs().max() / exact.abs().max()).item()
    print(f"f32b R={R} n_out={n_out} k_in={k_in}: rel err {e:.2e} (two-GEMM path {r:.2e})", flush=True)
    return e < 4 * r + 1e-6, fn, lambda: (gemm_ex(A_MN | B_MN, n_out, k_in, R, hi, lo, n_out, xs3, xs3.stride(0)),
                                          gemm_ex(A_MN | B_MN, n_out, k_in, R, hi, None, n_out, xs3[:, kp:], xs3.stride(0)))


for case in [(1024, 512, 384), (4096, 600, 200), (25600, 1024, 784)]:
    good, fn, two = check_f32b(*case)
    ok = good and ok
print("config-3 weight gradient: f32b %.1f us, two GEMMs %.1f us" % (timeit(fn), timeit(two)))
print("OK" if ok else "MISMATCH")
