import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import golden
from paper_2601_21407_b200 import network as N
cuda = torch.device('cuda', 0)
g = golden("cortex_small"); topo = N.build_network(float(g["scale"]), int(g["seed"]))
cfg = N.REST_CONFIG
for dtype in (np.float32, np.float64):
    a = N.CortexNetwork(topo, cfg, device=cuda, dtype=dtype, background="philox", seed=3)
    b = N.CortexNetwork(topo, cfg, device=cuda, dtype=dtype, background="philox", seed=3)
    b.t_dev.fill_(0)
    first = None
    for k in range(250):
        ra = a.step().clone()
        b._step_dev(); b.t += 1
        if not torch.equal(ra, b.gwords) or not torch.equal(a.v, b.v):
            first = k; break
    print(dtype.__name__, "eager device-t: first mismatch", first, "t_dev", int(b.t_dev.item()))
    a = N.CortexNetwork(topo, cfg, device=cuda, dtype=dtype, background="philox", seed=3)
    b = N.CortexNetwork(topo, cfg, device=cuda, dtype=dtype, background="philox", seed=3)
    first = None
    for k in range(120):
        ra = a.step().clone()
        rec = torch.empty((1, b.words_global), dtype=torch.int32, device=cuda)
        b.advance(1, steps_per_graph=1, record=rec)
        if not torch.equal(ra, rec[0]) or not torch.equal(a.v, b.v):
            first = k; break
    print(dtype.__name__, "graph S=1: first mismatch", first)
