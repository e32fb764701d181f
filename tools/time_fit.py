"""Time learn.fit on the reference's default teacher-student task (bench leg)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
print(json.dumps(bench.readout_fit_leg(torch, dev, epochs=int(sys.argv[1]) if len(sys.argv) > 1 else 20)))
