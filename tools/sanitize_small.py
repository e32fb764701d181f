"""Small-shape runs of the kernels with hand-rolled synchronisation, for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_small.py net|bwd|gemm|fwd

net  -- the persistent cooperative network kernel hh_net (grid barrier,
        cp.async ring prefetch, shared-memory delivery lists), 40 steps of the
        small golden network, with and without the thalamic drive
bwd  -- the BPTT kernel hh_bwd2 (cp.async shared-memory operand ring) and the
        training forward, through one HHLayer.mse_loss step (B 4 x 64 x T 24)
gemm -- k_umma_gemm_2sm (CTA pair, TMA, mbarriers, TMEM) and the 1-SM
        persistent k_umma_gemm_p, plain and dual-A, K- and MN-major operands
fwd  -- the fused-stimulus forward hh_fwdp_v4 (config-2 channel set, 4096 x 64)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

which = sys.argv[1]
dev = torch.device("cuda", 0)

if which == "net":
    from paper_2601_21407_b200 import network as N
    g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                             "cortex_small.npz"))
    topo = N.build_network(float(g["scale"]), int(g["seed"]))
    net = N.CortexNetwork(topo, N.REST_CONFIG, device=dev, dtype=np.float32, background="philox", seed=1)
    assert net.persistent_ok()
    net.advance(40)
    cfg = N.THALAMIC_CONFIG
    thal = {"t_on_ms": 0.5, "duration_ms": 2.0, "rate_hz": 400.0, "weight": cfg.bg_mean, "weight_std": cfg.bg_std}
    tt = N._thalamic_setup(topo, thal, 4.0, cfg.dt, np.random.default_rng(3))
    net2 = N.CortexNetwork(topo, cfg, device=dev, dtype=np.float32, background="philox", seed=2)
    net2.set_thalamic(*tt)
    net2.advance(40)
elif which == "bwd":
    from paper_2601_21407_b200.layer import HHLayer
    torch.manual_seed(0)
    for budget in (None, 4):
        layer = HHLayer(32, 64, w_mean=0.5, w_std=0.3, device=dev, budget=budget)
        x = ((torch.rand((24, 4, 32), device=dev) < 0.3).float()).requires_grad_(True)
        layer.mse_loss(x).backward()
        v, s = layer(x)
        ((v * v).mean() + s.sum() * 1e-3).backward()
elif which == "gemm":
    from paper_2601_21407_b200 import layer as L
    torch.manual_seed(0)
    for (M, N, K) in ((1024, 256, 128), (256, 96, 64)):       # CTA-pair path, then the 1-SM path
        a = torch.randn((M, K), device=dev).to(torch.bfloat16)
        b = torch.randn((N, K), device=dev).to(torch.bfloat16)
        out = L.gemm(a, b, K)
        ref = a.float() @ b.float().t()
        assert torch.allclose(out, ref, rtol=1e-2, atol=1e-2)
        lo = torch.randn((M, K), device=dev).to(torch.bfloat16)
        out2 = L.gemm_ex(0, M, N, K, a, lo, K, b, K)
        assert torch.allclose(out2, (a.float() + lo.float()) @ b.float().t(), rtol=1e-2, atol=1e-2)
        at = a.t().contiguous()                              # MN-major A
        out3 = L.gemm_ex(L.A_MN, M, N, K, at, None, M, b, K)
        assert torch.allclose(out3, ref, rtol=1e-2, atol=1e-2)
elif which == "fwd":
    from paper_2601_21407_b200 import defaults as DF
    from paper_2601_21407_b200.population import PoissonCurrent, Population
    p = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
    pop = Population(p, 4096, chunk=32, device=dev)
    pop.advance(PoissonCurrent(2.0, 2.0, seed=1), 64)
else:
    raise SystemExit(f"unknown {which}")
torch.cuda.synchronize()
print("ok", which)
