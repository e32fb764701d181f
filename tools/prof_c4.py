"""Config-4 training steps (bench c4_leg) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
r = bench.c4_leg(torch, dev)
print(r["ms_per_step"])
