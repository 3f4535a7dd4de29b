"""Host SAH build vs device LBVH build: build time and the trace speed each
tree gives (full frames, CUDA events).

    python tools/bvh_device_bench.py [c2 c3 c5]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import _lib, propagation, workloads  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402
from tools.probe_trace import time_trace  # noqa: E402


def main(names):
    for name in names:
        w = workloads.WORKLOADS[name]()
        row = {}
        for build in ("host", "device"):
            sc = scene_from_workload(w, bvh_build=build)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sc._device_handle()
            torch.cuda.synchronize()
            create_s = time.perf_counter() - t0
            cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces,
                                          sh_order=w.order, bin_s=w.bin_s, n_bins=w.n_bins,
                                          listener_radius=w.radius, seed=w.seed)
            n_src = min(len(w.sources), 32)
            tr = propagation.FrameTracer(sc, n_src, cfg)
            tr.set_sources(w.sources[:n_src])
            ms, segs = time_trace(tr, w, reps=10)
            st = tr.trace_stats()
            nodes = sum(s.nodes_visited for s in st)
            tris = sum(s.triangles_tested for s in st)
            info = sc.device_info()
            row[build] = (create_s, ms, segs, nodes / max(segs, 1), tris / max(segs, 1), info)
            print(f"[{name}] {build:6s} create {create_s*1e3:9.1f} ms  nodes {info['n_nodes']:8d} "
                  f"depth {info['max_depth']:3d}  frame {ms*1e3:9.1f} us  {segs/ms/1e6:6.3f} Gseg/s  "
                  f"nodes/seg {nodes/max(segs,1):6.2f} tris/seg {tris/max(segs,1):6.2f}", flush=True)
            if build == "device":
                # rebuild alone (device arrays already resident), CUDA events
                t = _lib.torch()
                dv = [_lib.to_device(a, t.float64) for a in (sc.v0, sc.e1, sc.e2, sc.normals)]
                ts = []
                for _ in range(6):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record()
                    _lib.check(_lib.lib().ef_scene_rebuild(sc._handle, *[_lib.ptr(x) for x in dv],
                                                           _lib.stream_handle()))
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                print(f"[{name}] device rebuild {np.median(ts[1:]):.3f} ms (median of 5; "
                      f"{len(sc.v0)} triangles)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c5"])
