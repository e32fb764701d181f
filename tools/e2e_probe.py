"""Break down the host-buffer (e2e) path: PCIe and host-copy bandwidths on this
box, then repeated dynamics.simulate(numpy) calls at the bench size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_21407_b200 import _pipeline
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200 import dynamics as Dy

dev = torch.device("cuda", 0)
N = 1 << 28  # 1 GiB of fp32
host_p = torch.empty(N, dtype=torch.float32, pin_memory=True)
host_u = torch.empty(N, dtype=torch.float32)
d = torch.empty(N, dtype=torch.float32, device=dev)


def bw(fn, nbytes, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9


print("H2D pinned   %.1f GB/s" % bw(lambda: d.copy_(host_p, non_blocking=True), 4 * N))
print("D2H pinned   %.1f GB/s" % bw(lambda: host_p.copy_(d, non_blocking=True), 4 * N))
print("H2D pageable %.1f GB/s" % bw(lambda: d.copy_(host_u), 4 * N))
print("D2H pageable %.1f GB/s" % bw(lambda: host_u.copy_(d), 4 * N))
a = np.ones(N, dtype=np.float32)
b = host_p.numpy()
print("host copy 1 thread  %.1f GB/s" % bw(lambda: np.copyto(b, a), 4 * N))
print("host copy threaded  %.1f GB/s" % bw(lambda: _pipeline._par_copy(b.reshape(256, -1), a.reshape(256, -1)), 4 * N))
t = time.perf_counter()
x = _pipeline.pinned_empty((20, 10_000_000), np.float64)
print("pinned alloc 1.6 GB: %.3f s" % (time.perf_counter() - t))
del x, host_p, host_u, d, a, b

p = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
i = (2.0 * np.random.default_rng(0).poisson(2.0, size=(20, 10_000_000))).astype(np.float32)
for k in range(4):
    t = time.perf_counter()
    tr = Dy.simulate(p, i)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    print("simulate(numpy 20 x 1e7) call %d: %.3f s -> %.3e neuron-steps/s" % (k, el, 2e8 / el))
    del tr
