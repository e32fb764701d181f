"""Run the config-1 bench leg alone."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

print(json.dumps(bench.c1_leg(torch, torch.device("cuda", 0))))
