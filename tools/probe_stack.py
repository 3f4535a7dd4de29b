"""Traversal-stack overflow probe: pushes per segment and how many of them
land past the split stack's 6 shared entries (in local memory), for the
overlapping 50k-triangle soup of tests/test_gpu_parity.py and for C3 / C5.
Needs a profiling build whose probe depth is the shared depth:
    python tools/build_variant.py prof6 -DEF_PROFILE_PHASES -DEF_SPLIT_DEPTH_PROBE=6
    EF_LIB_PATH=paper_1803_00430_b200/libechoforge_b200_prof6.so python tools/probe_stack.py
Round 2 (one B200): soup 52.3 pushes per segment, 22.5 of them past the
shared top; C3 4.11 / 0.030; C5 2.85 / 0.024."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_1803_00430_b200 import _lib, propagation, workloads
from paper_1803_00430_b200.workloads import Workload
from paper_1803_00430_b200.scene import scene_from_workload
def soup():
    rng = np.random.default_rng(77)
    T = 50_000
    c = rng.uniform(0.0, 10.0, size=(T, 1, 3))
    tris = c + rng.normal(scale=0.5, size=(T, 3, 3))
    return Workload("soup50k", tris, rng.integers(0, 2, T).astype(np.int64),
                 np.array([[0.1, 0.2, 0.3, 0.4], [0.3, 0.2, 0.1, 0.05]]),
                 np.array([[0.5] * 4, [0.2, 0.4, 0.6, 0.8]]),
                 sources=np.array([[5.0, 5.0, 5.0], [1.0, 2.0, 8.0]]), listener=np.array([6.0, 4.0, 5.0]),
                 radius=0.5, n_rays=4096, max_bounces=24, order=2, seed=5)
for name, w, n in (("soup", soup(), 768), ("c3", workloads.WORKLOADS["c3"](), 4096), ("c5", workloads.WORKLOADS["c5"](), 4096)):
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, len(w.sources), cfg)
    tr.set_sources(w.sources)
    L = _lib.lib()
    L.ef_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
    out = np.zeros(24, np.uint64)
    tr.trace(w.listener, n_rays=n); torch.cuda.synchronize()
    L.ef_debug_phases(out.ctypes.data, 1)
    tr.trace(w.listener, n_rays=n); torch.cuda.synchronize()
    L.ef_debug_phases(out.ctypes.data, 1)
    na = float(out[9]); k = [float(out[12 + i]) / na for i in range(9)]
    print(f"{name}: lane-segments {na:.0f}; pushes per segment {k[0]:.2f}, of them past 6 shared entries {k[1]:.4f}; node visits {float(out[5])/na:.2f}")
