"""Host-side costs of the simulate(numpy) pipeline: staging copy, page-locking
the caller's array in place, H2D / D2H bandwidth, concurrent bidirectional."""
import time

import numpy as np
import torch

import sys
sys.path.insert(0, ".")
from paper_2601_21407_b200 import _pipeline as P

dev = torch.device("cuda", 0)
n = 10_000_000
a = (np.random.default_rng(0).random((20, n)) * 4).astype(np.float32)   # 800 MB pageable
st = torch.empty((6, n), dtype=torch.float32, pin_memory=True).numpy()
for k in range(2):
    t = time.perf_counter(); P._par_copy(st, a[:6]); dt = time.perf_counter() - t
print(f"staging copy 240 MB (16 threads): {dt*1e3:.1f} ms = {240e6/dt/1e9:.1f} GB/s")
t = time.perf_counter(); np.copyto(st, a[:6]); dt = time.perf_counter() - t
print(f"staging copy 240 MB (1 thread): {dt*1e3:.1f} ms")
cr = torch.cuda.cudart()
t = time.perf_counter()
rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
dt = time.perf_counter() - t
print(f"cudaHostRegister 800 MB: rc={rc} {dt*1e3:.1f} ms")
ta = torch.from_numpy(a)
d = torch.empty((20, n), dtype=torch.float32, device=dev)
for k in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(ta, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"H2D 800 MB from registered: {dt*1e3:.1f} ms = {0.8/dt:.1f} GB/s")
t = time.perf_counter(); cr.cudaHostUnregister(a.ctypes.data); dt = time.perf_counter() - t
print(f"cudaHostUnregister: {dt*1e3:.1f} ms")
o = torch.empty((20, n), dtype=torch.float64, pin_memory=True)
d64 = torch.empty((20, n), dtype=torch.float64, device=dev)
for k in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); o.copy_(d64, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"D2H 1.6 GB to pinned: {dt*1e3:.1f} ms = {1.6/dt:.1f} GB/s")
pi = torch.empty((20, n), dtype=torch.float32, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for k in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(pi, non_blocking=True)
    with torch.cuda.stream(s2):
        o.copy_(d64, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"bidirectional 0.8 GB H2D + 1.6 GB D2H: {dt*1e3:.1f} ms")
