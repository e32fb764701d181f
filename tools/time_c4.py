"""Config-4 training step: per-launch CUDA-event times of every layer component
(layer.TIMERS), median over 7 eager steps -- which layer each kernel time
belongs to (the bench reports the per-component sums)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_21407_b200 import layer as L
from paper_2601_21407_b200.layer import HHLayer

dev = torch.device("cuda", 0)
B, T = 256, 100
torch.manual_seed(1)
ov = os.environ.get("OVERLAP", "1") == "1"
net = torch.nn.ModuleList([
    HHLayer(784, 2048, w_mean=0.05, w_std=0.1, check_finite=False, device=dev, outputs="spikes", overlap_weight_grad=ov),
    HHLayer(2048, 2048, w_mean=0.3, w_std=0.1, check_finite=False, device=dev, outputs="spikes", overlap_weight_grad=ov),
    HHLayer(2048, 10, w_mean=0.3, w_std=0.1, check_finite=False, device=dev, outputs="v", overlap_weight_grad=ov)])
g = torch.Generator(device=dev).manual_seed(1)
x = (torch.rand((T, B, 784), device=dev, generator=g) < 0.2).float() + 0.1 * torch.randn((T, B, 784), device=dev, generator=g)
y = torch.randint(0, 10, (B,), device=dev, generator=g)


def step():
    for p in net.parameters():
        p.grad = None
    h = x
    for lyr in net[:-1]:
        _, h = lyr(h)
    v, _ = net[-1](h)
    torch.nn.functional.cross_entropy(v.mean(0), y).backward()


for _ in range(3):
    step()
reps = 7
torch.cuda.synchronize()
L.TIMERS = {}
for _ in range(reps):
    step()
torch.cuda.synchronize()
recs, L.TIMERS = L.TIMERS, None
for name, rr in recs.items():
    per = len(rr) // reps
    cols = []
    for k in range(per):
        ts = sorted(rr[r * per + k][0].elapsed_time(rr[r * per + k][1]) for r in range(reps))
        cols.append(round(ts[reps // 2] * 1e3, 1))
    print(f"{name:14s} per launch (us, in call order): {cols}")
