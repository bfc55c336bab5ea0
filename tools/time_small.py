"""Timing aid for A/B builds (TCS_LIB_PATH): bench.py's small configs (C1
SpMM / C2 SDDMM, FP16 + TF32, CUDA-graph replays of 200 calls), the us per
call only; repeated `reps` times to show the spread."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    r = bench.small_configs(torch.device("cuda", 0))
    print(json.dumps({k: v for k, v in r.items() if k.endswith("_us")}))
