"""Config-3 training step (bench fwd_bwd leg) timing with per-kernel CUDA-event
times -- for A/B runs of kernel variants (env knobs such as HHB_JIT_BWD2_MINB).

    python tools/time_c3.py [bf16|bf16x3] ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

dev = torch.device("cuda", 0)
for proj in (sys.argv[1:] or ["bf16"]):
    r = bench.fwd_bwd_leg(torch, dev, proj, mufu_peak=4.63e12)
    k = r["roofline"]["kernels_ms_per_step"]
    print(json.dumps({"proj": proj, "env": {e: os.environ[e] for e in os.environ if e.startswith("HHB_")},
                      "ms_per_step": round(r["ms_per_step"], 4),
                      "kernels_us": {n: round(v * 1e3, 1) for n, v in k.items()}}))
