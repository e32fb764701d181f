"""Drive the config-3 training forward (fused MSE path) for an ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_21407_b200.layer import HHLayer

dev = torch.device("cuda", 0)
torch.manual_seed(0)
layer = HHLayer(784, 1024, w_mean=0.05, w_std=0.1, check_finite=False, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
x = ((torch.rand((100, 256, 784), device=dev, generator=g) < 0.2).float()
     + 0.1 * torch.randn((100, 256, 784), device=dev, generator=g))
for _ in range(3):
    layer.mse_loss(x).backward()
torch.cuda.synchronize()
print("ok")
