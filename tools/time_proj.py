"""The config-3 projection GEMM as the layer calls it (with / without bias)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_21407_b200.layer import gemm, to_bf16_padded

dev = torch.device("cuda", 0)
M, K, N = 25600, 784, 1024
x = torch.randn((M, K), device=dev)
w = torch.randn((N, K), device=dev)
b = torch.randn(N, device=dev)
xb, wb = to_bf16_padded(x), to_bf16_padded(w)
for name, f in (("no bias", lambda: gemm(xb, wb, K)), ("bias", lambda: gemm(xb, wb, K, bias=b)),
                ("cast x + gemm + bias", lambda: gemm(to_bf16_padded(x), wb, K, bias=b))):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    e1.synchronize()
    print(f"{name:24s} {e0.elapsed_time(e1) / 20 * 1e3:6.1f} us")
