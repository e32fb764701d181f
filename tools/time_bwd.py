"""CUDA-event timing of one hh_bwd launch at the config-3 shape (B=256 x 1024
neurons, T=100, RS, full storage) -- for A/B runs of backward variants."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2601_21407_b200 import adjoint as A, defaults as DF, dynamics as Dy
from paper_2601_21407_b200.dynamics import _forward

dev = torch.device("cuda", 0)
p = DF.cortical_rs_params(dt=0.1).with_(dtype=np.float32)
n, T = 256 * 1024, 100
K = int(os.environ.get("K", "1"))
g = torch.Generator(device=dev).manual_seed(0)
cur = 7.8 + 3.0 * torch.randn((T, n), device=dev, generator=g)
sv = 1e-4 * torch.randn((T, n), device=dev, generator=g)
s0 = Dy.init_state(p, (n,), device=dev)
nck = (T + K - 1) // K
ckpt = torch.empty((nck, 1 + p.n_gates, n), device=dev)
_forward(p, s0.v.clone(), s0.gates.clone(), cur, n, 1, T, ckpt=ckpt, ckpt_every=K)
hi = torch.empty((T, n), dtype=torch.bfloat16, device=dev)
lo = torch.empty_like(hi)
dsum = torch.zeros(n, device=dev)
spec = A.default_surrogate(p)
def run():
    adj_v = torch.zeros(n, device=dev)
    adj_g = torch.zeros((p.n_gates, n), device=dev)
    return A._backward(p, spec, cur, n, 1, T, n, ckpt, K, sv, None, adj_v, adj_g, want_d_i=False,
                       split=(hi, lo), d_sum=dsum)
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"bwd K={K} {os.environ.get('HHB_JIT_BWD_MINB', '-')} {ms:.3f} ms  {n * T / ms / 1e-3:.3e} neuron-steps/s")
