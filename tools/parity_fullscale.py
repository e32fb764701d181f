"""Config-2 parity at full scale: the float32 merged kernel (the bench path) vs
the float64 kernel (the reference's operation order, bit-close to NumPy) on
the same stimulus, 10M neurons x 10,000 steps.  Size-independent properties of
SURVEY §8 c3: per-neuron spike counts, first-spike steps (+-1), and V within
1e-4 |V64| + 0.02 mV for every neuron that has not spiked yet in either run.

    python tools/parity_fullscale.py [--neurons N] [--steps T]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200.dynamics import _forward, _unpack, init_state
from paper_2601_21407_b200.population import PoissonCurrent

ap = argparse.ArgumentParser()
ap.add_argument("--neurons", type=int, default=10_000_000)
ap.add_argument("--steps", type=int, default=10_000)
ap.add_argument("--chunk", type=int, default=100)
a = ap.parse_args()
dev = torch.device("cuda", 0)
n, T, C = a.neurons, a.steps, a.chunk
p32 = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
p64 = p32.with_(dtype=np.float64)
s32, s64 = init_state(p32, (n,), device=dev), init_state(p64, (n,), device=dev)
v32, g32 = s32.v.contiguous(), s32.gates.contiguous()
v64, g64 = s64.v.contiguous(), s64.gates.contiguous()
stim = PoissonCurrent(2.0, 2.0, seed=1234)
i32 = torch.empty((C, n), dtype=torch.float32, device=dev)
W = (n + 31) // 32
b32 = torch.empty((C, W), dtype=torch.int32, device=dev)
b64 = torch.empty((C, W), dtype=torch.int32, device=dev)
cnt32 = torch.zeros(n, dtype=torch.int32, device=dev)
cnt64 = torch.zeros(n, dtype=torch.int32, device=dev)
first32 = torch.full((n,), -1, dtype=torch.int64, device=dev)
first64 = torch.full((n,), -1, dtype=torch.int64, device=dev)
quiet = torch.ones(n, dtype=torch.bool, device=dev)       # no spike yet in either run
v_checked = 0
v_fail = 0
steps_idx = torch.arange(C, device=dev)[:, None]
t0 = time.time()
for c0 in range(0, T, C):
    tc = min(C, T - c0)
    stim.fill(i32[:tc], c0, 0)
    i64 = i32[:tc].double()
    _forward(p32, v32, g32, i32[:tc], n, 1, tc, v_fin=v32, g_fin=g32, bits=b32[:tc], step_base=c0)
    _forward(p64, v64, g64, i64, n, 1, tc, v_fin=v64, g_fin=g64, bits=b64[:tc], step_base=c0)
    del i64
    for bits, cnt, first in ((b32, cnt32, first32), (b64, cnt64, first64)):
        s = _unpack(bits[:tc], tc, n).to(torch.int32)
        cnt += s.sum(0, dtype=torch.int32)
        has = s.any(0)
        fidx = torch.where(s.bool(), steps_idx[:tc], C).min(0).values + c0
        first.copy_(torch.where((first < 0) & has, fidx, first))
        del s
    # V contract on the neurons still quiet in both runs at the chunk end
    q = quiet & (first32 < 0) & (first64 < 0)
    dv = (v32.double() - v64).abs()
    bound = 1e-4 * v64.abs() + 0.02
    v_checked += int(q.sum().item())
    v_fail += int((q & (dv > bound)).sum().item())
    quiet = q
torch.cuda.synchronize()
el = time.time() - t0
dc = (cnt32 - cnt64).abs()
both = (first32 >= 0) & (first64 >= 0)
res = {
    "neurons": n, "steps": T, "seconds": round(el, 1),
    "spikes_fp64_total": int(cnt64.sum().item()), "spikes_fp32_total": int(cnt32.sum().item()),
    "count_equal_frac": float((dc == 0).double().mean().item()),
    "count_diff_le1_frac": float((dc <= 1).double().mean().item()),
    "count_diff_max": int(dc.max().item()),
    "first_spike_both_frac": float(both.double().mean().item()),
    "first_spike_equal_frac_of_both": float(((first32 == first64) & both).double().sum().item() / max(1, int(both.sum().item()))),
    "first_spike_pm1_frac_of_both": float((((first32 - first64).abs() <= 1) & both).double().sum().item() / max(1, int(both.sum().item()))),
    "spiked_in_one_run_only": int(((first32 >= 0) ^ (first64 >= 0)).sum().item()),
    "prespike_v_checks": v_checked, "prespike_v_violations": v_fail,
}
print(json.dumps(res))
