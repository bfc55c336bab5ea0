"""Timing aid for A/B builds (TCS_LIB_PATH): bench.py's small configs (C1
SpMM / C2 SDDMM, FP16 + TF32, CUDA-graph replays of 200 calls), the us per
call only; repeated `reps` times to show the spread.  `floor_us`: the same
graph replay of a one-element torch kernel (per-node launch floor)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def floor_us(reps=200):
    x = torch.zeros(1, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        x.add_(1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            x.add_(1)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / reps, 2)


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    r = bench.small_configs(torch.device("cuda", 0))
    out = {k: v for k, v in r.items() if k.endswith("_us")}
    out["floor_us"] = floor_us()
    print(json.dumps(out))
