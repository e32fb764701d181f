"""Per-phase timing of the persistent kernel with R replicas per launch."""
import os
import sys

os.environ["HHB_NET_REPLICAS_PERSIST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_21407_b200 import network as N

dev = torch.device("cuda", 0)
topo = N.build_network(0.5, 0)
for R in [int(x) for x in sys.argv[1:]] or [1, 4]:
    rep = N.CortexReplicas(topo, N.REST_CONFIG, R, device=dev, dtype=np.float32, seed=1)
    rep.advance(200)
    steps = 300
    tiles = (rep.n_pad + 255) // 256
    rep.timing = torch.zeros((steps, tiles, 4), dtype=torch.int64, device=dev)
    rep.advance(steps)
    torch.cuda.synchronize()
    tm = rep.timing.cpu().numpy().astype(np.float64)
    st, sp, bp, dn = (tm[..., k] for k in range(4))
    t0 = st.min(axis=1)
    print(f"R={R}: step {np.median(np.diff(t0)) / 1e3:.2f} us; A {np.median((sp - st).mean(1)) / 1e3:.2f}/"
          f"{np.median((sp - st).max(1)) / 1e3:.2f}; barrier {np.median((bp - sp.max(1)[:, None]).mean(1)) / 1e3:.2f}; "
          f"B {np.median((dn - bp).mean(1)) / 1e3:.2f}/{np.median((dn - bp).max(1)) / 1e3:.2f}")
