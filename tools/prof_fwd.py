"""Small driver for ncu captures of the hot kernels (one GPU).

    python tools/prof_fwd.py [--neurons N] [--steps T] [--chunk C] [--bptt]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2601_21407_b200 import adjoint as A
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200 import dynamics as Dy
from paper_2601_21407_b200.population import PoissonCurrent, Population

ap = argparse.ArgumentParser()
ap.add_argument("--neurons", type=int, default=2_000_000)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--chunk", type=int, default=100)
ap.add_argument("--bptt", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
if a.bptt:
    p = DF.cortical_rs_params(dt=0.1).with_(dtype=np.float32)
    B, N, T = 256, 1024, 100
    i = 7.8 + 3.0 * torch.randn((T, B, N), device=dev)
    sv = torch.randn((T, B, N), device=dev) * 1e-4
    s0 = Dy.init_state(p, (B, N), device=dev)
    for _ in range(2):
        A.backward_through_time(p, s0, i, sv)
else:
    p = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
    pop = Population(p, a.neurons, chunk=a.chunk, device=dev)
    pop.advance(PoissonCurrent(2.0, 2.0, 1), a.steps, check=True)
torch.cuda.synchronize()
print("ok")
