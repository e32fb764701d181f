import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2601_21407_b200 import defaults as DF, dynamics as Dy
params = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
n, T = 10_000_000, 20
i_host = (2.0 * np.random.default_rng(0).poisson(2.0, size=(T, n))).astype(np.float32)
tr = Dy.simulate(params, i_host); del tr
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tr = Dy.simulate(params, i_host); torch.cuda.synchronize()
    print(f"total {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del tr
