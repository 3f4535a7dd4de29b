"""Render a few C4 blocks for S sources (profiling helper)."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import render, workloads  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
base = workloads.c4_params(n_sources=64)
import numpy as np  # noqa: E402
reps = (S + 63) // 64
p = {k: (np.concatenate([v] * reps)[:S] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == 64 else v)
     for k, v in base.items()}
r = render.SHRenderer(p)
x = torch.randn((S, 512), dtype=torch.float32, device="cuda") * 0.1
for _ in range(6):
    r.process(x, want_bus=False)
torch.cuda.synchronize()
print("ok", S)
