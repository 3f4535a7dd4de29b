"""Cycle phases of the analysis kernel's first CTA (needs the profiling
build: EF_LIB_PATH=..._prof.so):  python tools/probe_analysis.py [config]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import _lib, propagation, workloads  # noqa: E402
from paper_1803_00430_b200.analysis import Analyzer  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = workloads.WORKLOADS[name]()
sc = scene_from_workload(w)
cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                              bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
tr = propagation.FrameTracer(sc, len(w.sources), cfg)
tr.set_sources(w.sources)
tr.trace(w.listener)
an = Analyzer(len(w.sources), w.n_bins, sc.n_bands, w.order, w.bin_s)
L = _lib.lib()
L.ef_debug_analysis_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = np.zeros(7, np.uint64)
for _ in range(5):
    an.run(tr.H, tr.Dir, tr.stats, tr.sum_t)
torch.cuda.synchronize()
L.ef_debug_analysis_phases(out.ctypes.data, 1)
for _ in range(20):
    an.run(tr.H, tr.Dir, tr.stats, tr.sum_t)
torch.cuda.synchronize()
L.ef_debug_analysis_phases(out.ctypes.data, 0)
n = max(int(out[3]), 1)
print(f"[{name}] analysis CTA 0, cycles per call: start->pass1 {int(out[4]) / n:.0f}, pass 1 "
      f"{int(out[0]) / n:.0f} (rows done {int(out[5]) / n:.0f}, warp sums done {int(out[6]) / n:.0f}), "
      f"fit {int(out[1]) / n:.0f}, directivity+loudness {int(out[2]) / n:.0f}")
