"""Probe where the C2 frame time goes: vary the bounce cap (tail) and the
ray count (bulk) and time ef_trace alone with CUDA events.

    python tools/probe_trace.py [config]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import propagation, workloads  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402


def time_trace(tr, w, reps=20, **kw):
    for _ in range(3):
        tr.trace(w.listener, **kw)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record()
        tr.trace(w.listener, **kw)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    segs = int(tr.stats[:, 1].sum())
    return float(np.median(ts)), segs


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    w = workloads.WORKLOADS[name]()
    sc = scene_from_workload(w)
    print("scene", sc.device_info())
    for mb in (1, 2, 5, 10, 20, 50, 100):
        cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=mb, sh_order=w.order,
                                      bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius,
                                      seed=w.seed)
        tr = propagation.FrameTracer(sc, len(w.sources), cfg)
        tr.set_sources(w.sources)
        ms, segs = time_trace(tr, w)
        print(f"max_bounces {mb:4d}: {ms*1e3:8.1f} us  segs {segs:9d}  {segs/ms/1e6:7.3f} Gseg/s")
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    for mult in (1, 2, 4, 8, 16):
        tr = propagation.FrameTracer(sc, len(w.sources), cfg)
        tr.set_sources(w.sources)
        ms, segs = time_trace(tr, w, n_rays=w.n_rays * mult)
        print(f"rays x{mult:3d}: {ms*1e3:8.1f} us  segs {segs:9d}  {segs/ms/1e6:7.3f} Gseg/s")


if __name__ == "__main__" and len(sys.argv) <= 2:
    main()


def timing(name="c2"):
    """Per-path start/end (globaltimer ns) of one full frame."""
    w = workloads.WORKLOADS[name]()
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, len(w.sources), cfg, record=2)
    tr.set_sources(w.sources)
    for _ in range(3):
        tr.trace(w.listener)
    torch.cuda.synchronize()
    rows = tr.path_ids.cpu().numpy().reshape(-1, w.max_bounces)[:, :6].astype(np.int64)
    t0 = (rows[:, 0] & 0xffffffff) | (rows[:, 1] << 32)
    t1 = (rows[:, 2] & 0xffffffff) | (rows[:, 3] << 32)
    base = t0.min()
    t0 = (t0 - base) / 1e3
    t1 = (t1 - base) / 1e3
    nseg = rows[:, 5]
    dur = t1 - t0
    print(f"[{name}] span {t1.max():.1f} us; last path start {t0.max():.1f} us; "
          f"paths done by: 50% {np.percentile(t1, 50):.1f} 90% {np.percentile(t1, 90):.1f} "
          f"99% {np.percentile(t1, 99):.1f} 99.9% {np.percentile(t1, 99.9):.1f} 100% {t1.max():.1f}")
    order = np.argsort(-t1)[:8]
    for i in order:
        print(f"  path {i}: start {t0[i]:.1f} end {t1[i]:.1f} dur {dur[i]:.1f} us nseg {nseg[i]} "
              f"({dur[i] / max(nseg[i], 1):.2f} us/seg) sm {rows[i, 4]}")
    full = tr.path_ids.cpu().numpy().reshape(-1, w.max_bounces)
    i = int(np.argmax(t1))
    seg_t = full[i, 6:6 + min(nseg[i], w.max_bounces - 6)] / 1e3 + t0[i]
    print("  longest path: absolute end time (us) of segments 1..:",
          " ".join(f"{x:.0f}" for x in seg_t[::5]), "(every 5th)")
    for k in (1, 2, 4, 10, 50):
        sel = nseg == k
        if sel.any():
            print(f"  nseg={k:3d}: n={sel.sum():6d} mean dur {dur[sel].mean():.2f} us "
                  f"({dur[sel].mean() / k:.2f} us/seg)")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "timing":
    timing(sys.argv[1])


def single(name="c2", src=6, ray=27707, reps=5):
    """One path alone on the GPU: in-kernel duration and per-segment latency."""
    w = workloads.WORKLOADS[name]()
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, 1, cfg, record=2)
    tr.set_sources(w.sources[src:src + 1], [src])
    for _ in range(reps):
        tr.trace(w.listener, ray_ids=[ray])
        torch.cuda.synchronize()
        r = tr.path_ids.cpu().numpy().reshape(-1)[:6].astype(np.int64)
        t0 = (r[0] & 0xffffffff) | (r[1] << 32)
        t1 = (r[2] & 0xffffffff) | (r[3] << 32)
        print(f"[{name}] single path src {src} ray {ray}: {(t1 - t0) / 1e3:.1f} us, nseg {r[5]}, "
              f"{(t1 - t0) / 1e3 / r[5]:.2f} us/seg")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "single":
    single(sys.argv[1])


def knobs(name="c2"):
    """Frame time and device work per segment for the current EF_BVH_* knobs."""
    w = workloads.WORKLOADS[name]()
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, len(w.sources), cfg)
    tr.set_sources(w.sources)
    ms, segs = time_trace(tr, w)
    st = tr.stats.sum(0).cpu().numpy()
    info = sc.device_info()
    print(f"[{name}] CI={os.environ.get('EF_BVH_CI', '2')} LEAF={os.environ.get('EF_BVH_MAXLEAF', '4')} "
          f"nodes={info['n_nodes']} depth={info['max_depth']} leafmax={info['max_leaf']}: "
          f"{ms*1e3:.1f} us  nodes/seg {st[7]/st[1]:.2f} tris/seg {st[8]/st[1]:.2f}")
    tr1 = propagation.FrameTracer(sc, 1, cfg, record=2)
    tr1.set_sources(w.sources[6:7], [6])
    tr1.trace(w.listener, ray_ids=[27707])
    torch.cuda.synchronize()
    r = tr1.path_ids.cpu().numpy().reshape(-1)[:6].astype(np.int64)
    t0 = (r[0] & 0xffffffff) | (r[1] << 32)
    t1 = (r[2] & 0xffffffff) | (r[3] << 32)
    st1 = tr1.stats.sum(0).cpu().numpy()
    print(f"    single long path: {(t1 - t0) / 1e3 / r[5]:.2f} us/seg, nodes/seg {st1[7]/st1[1]:.2f} "
          f"tris/seg {st1[8]/st1[1]:.2f}")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "knobs":
    knobs(sys.argv[1])


def phases(name="c2", src=6, ray=27707):
    """Cycle breakdown of one path (needs EF_LIB_PATH=..._prof.so).  Segments
    run by tail_kernel report the tail phases; their finish_segment splits
    into counters 0-2 (listener / shading record + draws / direction), which
    the BVH path uses for visits / leaf tests / pops."""
    import ctypes
    from paper_1803_00430_b200 import _lib
    L = _lib.lib()
    L.ef_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
    w = workloads.WORKLOADS[name]()
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, 1, cfg, record=2)
    tr.set_sources(w.sources[src:src + 1], [src])
    out = np.zeros(12, np.uint64)
    for rep in range(3):
        L.ef_debug_phases(out.ctypes.data, 1)
        tr.trace(w.listener, ray_ids=[ray])
        torch.cuda.synchronize()
        L.ef_debug_phases(out.ctypes.data, 1)
    segs = int(out[4])
    names = ["inner visits", "leaf tests", "pops after leaf", "shading"]
    print(f"[{name}] path src {src} ray {ray}: {segs} segments; cycles per segment:")
    for i, n in enumerate(names):
        print(f"   {n:16s} {int(out[i]) / max(segs, 1):9.0f}")
    for i, n in zip(range(8, 12), ["tail sweep", "tail reduction", "tail finish", "tail barrier"]):
        print(f"   {n:16s} {int(out[i]) / max(segs, 1):9.0f}")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "phases":
    phases(sys.argv[1])
