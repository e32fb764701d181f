"""Timeline of one simulate(numpy) pipelined call (CUPTI via torch.profiler)."""
import sys
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, ".")
from paper_2601_21407_b200 import defaults as DF, dynamics as Dy
params = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
n, T = 10_000_000, 20
i_host = (2.0 * np.random.default_rng(0).poisson(2.0, size=(T, n))).astype(np.float32)
tr = Dy.simulate(params, i_host); del tr
tr = Dy.simulate(params, i_host); del tr
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr = Dy.simulate(params, i_host); torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0) / 1e3:8.2f} {(e.time_range.end - e.time_range.start) / 1e3:7.2f} ms  "
          f"{e.name[:60]}")
