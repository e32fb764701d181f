"""Forward GEMM efficiency vs K (epilogue share shrinks as K grows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_21407_b200.layer import gemm, to_bf16_padded

dev = torch.device("cuda", 0)
M, N = 25600, 1024
for K in (784, 1568, 3136, 6272):
    xb = to_bf16_padded(torch.randn((M, K), device=dev))
    wb = to_bf16_padded(torch.randn((N, K), device=dev))
    for _ in range(3):
        gemm(xb, wb, K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gemm(xb, wb, K)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"K={K:5d}  {ms * 1e3:7.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s")
