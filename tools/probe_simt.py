"""SIMT cost of per-lane traversal lengths (profiling build,
EF_PROFILE_PHASES): for one frame of a config, the node visits and triangle
tests actually done vs 32 x the warp's longest traversal of each segment
round.  python tools/probe_simt.py c5 [rays_per_source]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import build  # noqa: E402

import torch  # noqa: E402

from paper_1803_00430_b200 import _lib, propagation, workloads  # noqa: E402

_lib.LIB_PATH = build.build(profile_phases=True)   # before the first _lib.lib()
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    w = workloads.WORKLOADS[name]()
    n = int(sys.argv[2]) if len(sys.argv) > 2 else w.n_rays
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, len(w.sources), cfg)
    tr.set_sources(w.sources)
    L = _lib.lib()
    L.ef_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
    out = np.zeros(24, np.uint64)
    tr.trace(w.listener, n_rays=n)
    torch.cuda.synchronize()
    L.ef_debug_phases(out.ctypes.data, 1)
    tr.trace(w.listener, n_rays=n)
    torch.cuda.synchronize()
    L.ef_debug_phases(out.ctypes.data, 1)
    sn, mn, mt, st, na = (float(out[i]) for i in (5, 6, 7, 8, 9))
    segs = int(tr.stats[:, 1].sum())
    print(f"{name}: {segs} segments, {na:.0f} lane-segments counted")
    print(f"  node visits {sn:.4g} ({sn / na:.2f} per segment); 32 x warp max {mn:.4g}: "
          f"SIMT efficiency of the node loop {sn / mn:.3f}")
    print(f"  triangle tests {st:.4g} ({st / na:.2f} per segment); 32 x warp max {mt:.4g}: "
          f"efficiency {st / mt:.3f}")
    k = [float(out[12 + i]) / na for i in range(9)]
    print(f"  stack per segment: pushes {k[0]:.2f} (past the shared top {k[1]:.3f}), pops taken {k[2]:.2f}, "
          f"culled {k[3]:.2f}; node visits hitting 0/1/2/3+ children {k[4]:.2f}/{k[5]:.2f}/{k[6]:.2f}/{k[7]:.2f}; "
          f"leaf visits {k[8]:.2f}")



if __name__ == "__main__":
    main()
