"""Single-GPU estimate of C5 strong scaling (NOT a multi-GPU measurement):
rank g of N traces rays [g R/N, (g+1) R/N) of every source with no
data-path exchange except the histogram splats (fused into the kernel;
C5 has ~200 arrivals per frame), so a frame on N GPUs takes about the
slowest shard's time.  This times every shard of N = 1, 2, 4, 8 alone on
one B200 (CUDA events, 3 frames each after 2 warm-up frames) and reports
T_1 / (N * max_g T_g).  python tools/scaling_estimate.py [config]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import distributed, propagation, workloads  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    w = workloads.WORKLOADS[name]()
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, len(w.sources), cfg)
    tr.set_sources(w.sources)
    t1 = None
    print(f"{name}: strong scaling from shard times on one GPU (estimate; 2 warm-up + 3 timed frames per shard)")
    for n in (1, 2, 4, 8):
        shard_ms = []
        for g in range(n):
            ray0, nr = distributed.shard_rays(w.n_rays, g, n)
            for _ in range(2):
                tr.trace(w.listener, ray0=ray0, n_rays=nr, total_rays=w.n_rays)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(3):
                tr.trace(w.listener, ray0=ray0, n_rays=nr, total_rays=w.n_rays)
            b.record()
            torch.cuda.synchronize()
            shard_ms.append(a.elapsed_time(b) / 3)
        tmax = max(shard_ms)
        if t1 is None:
            t1 = tmax
        print(f"  N={n}: shard ms min {min(shard_ms):.2f} max {tmax:.2f}  "
              f"speed-up {t1 / tmax:.2f}x  efficiency {t1 / (n * tmax):.3f}", flush=True)


if __name__ == "__main__":
    main()
