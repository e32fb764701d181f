"""Time the morphology leg alone, optionally after the config-5 leg."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
print(json.dumps({k: v for k, v in bench.morph_leg(torch, dev).items() if k != "config"}))
if len(sys.argv) > 1:
    r = bench.c5_leg(torch, dev)
    print(json.dumps({k: r[k] for k in ("value", "ms_per_network_step")}))
    print(json.dumps({k: v for k, v in bench.morph_leg(torch, dev).items() if k != "config"}))
