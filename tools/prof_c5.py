"""Kernel-time breakdown of the config-5 network step (graph replay)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2601_21407_b200 import network as N
dev = torch.device("cuda", 0)
topo = N.build_network(0.5, 0)
net = N.CortexNetwork(topo, N.REST_CONFIG, device=dev, dtype=np.float32, background="philox", seed=1)
net.advance(256)
torch.cuda.synchronize()
steps = 640
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    net.advance(steps)
    torch.cuda.synchronize()
tot, cnt = collections.Counter(), collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name[:80]] += e.device_time_total
        cnt[e.name[:80]] += 1
print(f"kernel sum per step {sum(tot.values()) / steps:.2f} us")
for k, v in tot.most_common(10):
    print(f"{v / steps:8.2f} us  {cnt[k] / steps:4.1f}x  {k}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); net.advance(steps); e1.record(); e1.synchronize()
print(f"wall per step {e0.elapsed_time(e1) / steps * 1e3:.2f} us")
