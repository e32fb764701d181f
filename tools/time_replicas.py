"""Time the config-5 replicas leg (persistent vs graph path: HHB_NET_GRAPH=1)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

reps = tuple(int(x) for x in sys.argv[1:]) or (1, 4, 8, 16, 32, 64)
r = bench.c5_replicas_leg(torch, torch.device("cuda", 0), replicas=reps)
print(json.dumps({k: (round(v["ms_per_network_step"] * 1e3, 2), f'{v["value"]:.3g}') for k, v in r["by_replicas"].items()}))
