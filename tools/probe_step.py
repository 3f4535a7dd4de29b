"""Device time of the step's parts with CUDA events: trace alone, analysis
alone (on the same histogram), and the two back to back.

    python tools/probe_step.py [config]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import propagation, workloads  # noqa: E402
from paper_1803_00430_b200.analysis import Analyzer  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    w = workloads.WORKLOADS[name]()
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, len(w.sources), cfg)
    tr.set_sources(w.sources)
    an = Analyzer(len(w.sources), w.n_bins, sc.n_bands, w.order, w.bin_s)
    t_tr = timed(lambda: tr.trace(w.listener))
    t_an = timed(lambda: an.run(tr.H, tr.Dir, tr.stats, tr.sum_t))
    t_both = timed(lambda: (tr.trace(w.listener), an.run(tr.H, tr.Dir, tr.stats, tr.sum_t)))
    print(f"[{name}] trace {t_tr:.1f} us, analysis {t_an:.1f} us, step {t_both:.1f} us "
          f"(gap {t_both - t_tr - t_an:.1f} us)")


if __name__ == "__main__":
    main()
