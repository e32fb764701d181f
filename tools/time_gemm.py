"""CUDA-event timing of the layer GEMM shapes (config 3) through hhb_gemm_ex."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_21407_b200.layer import gemm_ex, A_MN, B_MN
dev = torch.device("cuda", 0)
T, B, K_in, N_out = 100, 256, 784, int(os.environ.get("NOUT", "1024"))
M = T * B
xb = torch.randn((M, K_in), device=dev).to(torch.bfloat16)
wb = torch.randn((N_out, K_in), device=dev).to(torch.bfloat16)
hi = torch.randn((M, N_out), device=dev).to(torch.bfloat16)
lo = (torch.randn((M, N_out), device=dev) * 1e-3).to(torch.bfloat16)
cases = {"fwd  I=X W^T": lambda: gemm_ex(0, M, N_out, K_in, xb, None, K_in, wb, K_in),
         "dW = dI^T X ": lambda: gemm_ex(A_MN | B_MN, N_out, K_in, M, hi, lo, N_out, xb, K_in),
         "dX = dI W   ": lambda: gemm_ex(B_MN, M, K_in, N_out, hi, lo, N_out, wb, K_in)}
for name, f in cases.items():
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    flop = 2.0 * M * N_out * K_in * (2 if "d" in name[:2] else 1)
    print(f"{name} {ms * 1e3:7.1f} us  {flop / ms / 1e9:7.1f} TFLOP/s")
