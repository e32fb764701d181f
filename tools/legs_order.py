"""Run the secondary bench legs in bench.py's order, timing each (isolation check)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
import gc
for name, fn in (("c1", bench.c1_leg), ("fwd_bwd", bench.fwd_bwd_leg), ("c4", bench.c4_leg), ("c5", bench.c5_leg),
                 ("morph", bench.morph_leg), ("morph2", bench.morph_leg)):
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    t = time.perf_counter()
    r = fn(torch, dev)
    print(name, f"{time.perf_counter() - t:.1f}s", json.dumps({k: r[k] for k in r if k in ("value", "ms_per_step")}),
          f"mem {torch.cuda.memory_reserved() / 1e9:.1f} GB reserved", flush=True)
