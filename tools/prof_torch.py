"""Kernel-time breakdown of the config-3 / config-4 training steps from the
CUDA activity trace (torch.profiler / CUPTI), i.e. in a normal concurrent run
(ncu serialises and cold-starts every kernel)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import bench

dev = torch.device("cuda", 0)
which = sys.argv[1] if len(sys.argv) > 1 else "c3"
leg = bench.fwd_bwd_leg if which == "c3" else bench.c4_leg
leg(torch, dev)   # warm (includes its own timing)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = leg(torch, dev)
steps = 3 + (10 if which == "c3" else 5)
tot = collections.Counter()
cnt = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name[:70]] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name[:70]] += 1
allt = sum(tot.values())
print(f"{which}: {r['ms_per_step']:.3f} ms/step (events); kernel sum per step {allt / steps / 1e3:.3f} ms")
for k, v in tot.most_common(25):
    print(f"{v / steps:9.1f} us  {cnt[k] / steps:5.1f}x  {k}")
