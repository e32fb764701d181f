"""Time the config-5 leg (and the replicas leg) alone."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
r = bench.c5_leg(torch, dev)
print(json.dumps({k: r[k] for k in ("value", "ms_per_network_step")}))
