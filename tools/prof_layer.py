"""One config-3 layer training step (after warm-up) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_21407_b200.layer import HHLayer
dev = torch.device("cuda", 0)
torch.manual_seed(0)
layer = HHLayer(784, 1024, w_mean=0.05, w_std=0.1, device=dev, proj=os.environ.get("PROJ", "bf16"))
x = ((torch.rand((100, 256, 784), device=dev) < 0.2).float() + 0.1 * torch.randn((100, 256, 784), device=dev))   # data: no input gradient (bench fwd_bwd)
for _ in range(int(os.environ.get("STEPS", "3"))):
    layer.zero_grad(set_to_none=True)
    layer.mse_loss(x).backward()        # the bench's fused-MSE step (fwd_bwd)
torch.cuda.synchronize()
print("ok")
