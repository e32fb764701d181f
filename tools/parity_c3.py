"""Config-3 gradient parity at the full shape: HHLayer (bf16 tcgen05 projection,
float32 merged HH kernels, bf16x2 gradient GEMMs, fused MSE) against the
float64 kernels (the reference's operation order) on the same bf16-rounded
operands: dW, db, dX, d_c_m, d_g_max normwise relative errors (contract 1e-3,
SURVEY §8 c3b).  --unrounded compares against the reference composition on the
UNROUNDED float64 x and W (learn.py:210-211 computes in float64); the layer's
projection precision is --proj (bf16 | bf16x3).

    python tools/parity_c3.py [--batch B] [--steps T] [--unrounded] [--proj bf16x3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_21407_b200 import adjoint as A
from paper_2601_21407_b200 import dynamics as Dy
from paper_2601_21407_b200.defaults import cortical_rs_params
from paper_2601_21407_b200.layer import HHLayer

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--n-in", type=int, default=784)
ap.add_argument("--n-out", type=int, default=1024)
ap.add_argument("--unrounded", action="store_true")
ap.add_argument("--proj", default="bf16")
a = ap.parse_args()
dev = torch.device("cuda", 0)
B, T, K, N = a.batch, a.steps, a.n_in, a.n_out
torch.manual_seed(0)
layer = HHLayer(K, N, w_mean=0.05, w_std=0.1, device=dev, proj=a.proj)
g = torch.Generator(device=dev).manual_seed(0)
x = ((torch.rand((T, B, K), device=dev, generator=g) < 0.2).float()
     + 0.1 * torch.randn((T, B, K), device=dev, generator=g)).requires_grad_(True)
loss = layer.mse_loss(x)
loss.backward()

# float64 reference on the same bf16-rounded operands (or the unrounded ones)
if a.unrounded:
    xb = x.detach().double()
    wb = layer.weight.detach().double()
else:
    xb = x.detach().to(torch.bfloat16).double()
    wb = layer.weight.detach().to(torch.bfloat16).double()
drive = (xb @ wb.t() + layer.bias.detach().double()).reshape(T, B * N).contiguous()
p64 = cortical_rs_params(dt=0.1)
tr = Dy.simulate(p64, drive)
v = tr.v_series
seed = 2.0 * v / v.numel()
res = A.backward_through_time(p64, Dy.init_state(p64, (B * N,), device=dev), drive, seed)
d_drive = res.d_i.reshape(T * B, N)
dW = d_drive.t() @ xb.reshape(T * B, K)
db = d_drive.sum(0)
dX = (d_drive @ wb).reshape(T, B, K)


def nrel(a_, b_):
    return float((a_.double() - b_).norm() / b_.norm())


pg = layer.param_grads.cpu().numpy()
v32 = layer(x.detach())[0].reshape(T, B * N).double()
spk32 = layer(x.detach())[1].reshape(T, B * N).bool()
out = {"batch": B, "steps": T, "n_in": K, "n_out": N, "unrounded": a.unrounded, "proj": a.proj,
       "spike_count_mismatch_neurons": int((spk32.sum(0) != tr.spike_series.sum(0)).sum().item()),
       "v_maxabs": float((v32 - v).abs().max().item()),
       "loss_rel": abs(float(loss.item()) - float((v * v).mean().item())) / float((v * v).mean().item()),
       "dW": nrel(layer.weight.grad, dW), "db": nrel(layer.bias.grad, db), "dX": nrel(x.grad, dX),
       "d_c_m": abs(pg[0] - res.d_c_m) / abs(res.d_c_m),
       "d_g_max": float(np.linalg.norm(pg[1:] - res.d_g_max) / np.linalg.norm(res.d_g_max))}
print(json.dumps(out))
