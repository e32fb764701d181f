"""Drive the persistent network kernel once for an ncu capture (config 5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_21407_b200 import network as N

dev = torch.device("cuda", 0)
topo = N.build_network(float(os.environ.get("SCALE", "0.5")), 0)
net = N.CortexNetwork(topo, N.REST_CONFIG, device=dev, dtype=np.float32, background="philox", seed=1)
net.advance(200)
net.advance(int(os.environ.get("STEPS", "400")))
torch.cuda.synchronize()
print("ok", net.t)
# per-phase timing of one recorded run: net.timing = [steps][tiles][4] globaltimer stamps
steps = 300
tiles = (net.n + 255) // 256
net.timing = torch.zeros((steps, tiles, 4), dtype=torch.int64, device=dev)
net.advance(steps)
torch.cuda.synchronize()
tm = net.timing.cpu().numpy().astype(np.float64)
net.timing = None
st, sp, bp, dn = (tm[..., k] for k in range(4))
t0 = st.min(axis=1)
arrive_last = sp.max(axis=1)
print(f"per step (us, median over steps): total {np.median(np.diff(t0)) / 1e3:.2f}")
print(f"  phase A (input+HH, mean / max block): {np.median((sp - st).mean(1)) / 1e3:.2f} / {np.median((sp - st).max(1)) / 1e3:.2f}")
print(f"  barrier: last arrival -> release (mean block): {np.median((bp - arrive_last[:, None]).mean(1)) / 1e3:.2f}")
print(f"  barrier wait incl. imbalance (mean block): {np.median((bp - sp).mean(1)) / 1e3:.2f}")
print(f"  phase B (delivery, mean / max block): {np.median((dn - bp).mean(1)) / 1e3:.2f} / {np.median((dn - bp).max(1)) / 1e3:.2f}")
print(f"  start skew (max - min block start): {np.median(st.max(1) - st.min(1)) / 1e3:.2f}")
