"""simulate(numpy) for config 1 (1,024 x 10,000 squid, float32 I): the host-buffer path alone."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_21407_b200 import defaults as DF  # noqa: E402
from paper_2601_21407_b200 import dynamics as Dy  # noqa: E402

p = DF.squid_axon_params(dt=0.01).with_(dtype=np.float32)
i = np.full((10000, 1024), 10.0, dtype=np.float32)
for _ in range(3):
    Dy.simulate(p, i)
torch.cuda.synchronize()
ts = []
for _ in range(25):
    t0 = time.perf_counter()
    tr = Dy.simulate(p, i)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    del tr
ts.sort()
print(f"c1 simulate(numpy): min {ts[0] * 1e3:.2f} ms  median {ts[len(ts) // 2] * 1e3:.2f} ms  "
      f"({1024 * 10000 / ts[len(ts) // 2]:.3e} neuron-steps/s at the median)")
