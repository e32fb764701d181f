"""Kernel-time breakdown of one learn.fit epoch (CUPTI via torch.profiler)."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2601_21407_b200 import learn as L

task = L.make_teacher_student_task()
L.fit(L.make_student(task), task, L.TrainConfig(epochs=3))
E = 5
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    L.fit(L.make_student(task), task, L.TrainConfig(epochs=E))
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / E
tot, cnt = collections.Counter(), collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name[:80]] += e.device_time_total
        cnt[e.name[:80]] += 1
print(f"wall {wall:.3f} ms/epoch (under profiler); kernel sum {sum(tot.values()) / E / 1e3:.3f} ms/epoch, "
      f"{sum(cnt.values()) / E:.0f} launches/epoch")
for k, v in tot.most_common(30):
    print(f"{v / E:9.1f} us  {cnt[k] / E:5.1f}x  {k}")
