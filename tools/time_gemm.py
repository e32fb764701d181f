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
from paper_2601_21407_b200 import _native as nat
from paper_2601_21407_b200.layer import _workspace
x32 = torch.randn((M, K_in), device=dev)
w32 = torch.randn((N_out, K_in), device=dev)
out32 = torch.empty((M, N_out), device=dev)


def tf32_fwd():
    lib = nat.load()
    ws_n = int(lib.hhb_gemm_workspace(M, N_out, 32))
    ws = _workspace(ws_n, dev) if ws_n else None
    nat.check(lib.hhb_gemm(1, M, N_out, K_in, x32.data_ptr(), K_in, w32.data_ptr(), K_in, None, out32.data_ptr(),
                           N_out, 0, None if ws is None else ws.data_ptr(), torch.cuda.current_stream().cuda_stream),
              "tf32")


cases = {"fwd  I=X W^T": lambda: gemm_ex(0, M, N_out, K_in, xb, None, K_in, wb, K_in),
         "fwd  tf32 (fp32 X, W read directly)": tf32_fwd,
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
