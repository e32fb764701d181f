"""Time the e2e leg (simulate(numpy) with host buffers) alone."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2601_21407_b200 import defaults as DF  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--neurons", type=int, default=10_000_000)
ap.add_argument("--e2e-steps", type=int, default=20)
a = ap.parse_args()
params = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=__import__("numpy").float32)
r = bench.e2e_leg(torch, a, params, 0)
print(json.dumps({k: r[k] for k in ("value", "seconds_per_step")}))
