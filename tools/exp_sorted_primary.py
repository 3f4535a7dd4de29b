"""Experiment: do direction-sorted primary rays (coherent warps) trace
faster?  C5 scene, one source at a time, 2^20 rays: natural ray order vs the
same rays ordered by an octahedral direction cell (Morton), via ray_ids."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1803_00430_b200 import propagation, workloads  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402


def dirs_of(seed, src, n):
    out = np.zeros((n, 3))
    for r in range(n):
        out[r] = O.sample_sphere(seed, src, r, 0)
    return out


def cell_key(d, bits=8):
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    s = np.abs(x) + np.abs(y) + np.abs(z)
    u, v = x / s, y / s
    neg = z < 0
    u2 = np.where(neg, (1 - np.abs(v)) * np.sign(u), u)
    v2 = np.where(neg, (1 - np.abs(u)) * np.sign(v), v)
    qu = np.clip(((u2 + 1) * 0.5 * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    qv = np.clip(((v2 + 1) * 0.5 * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros_like(qu)
    for b in range(bits):
        key |= ((qu >> b) & 1) << (2 * b) | ((qv >> b) & 1) << (2 * b + 1)
    return key


def main():
    w = workloads.c5_city_grid()
    sc = scene_from_workload(w)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    for s in (0, 77, 201):
        tr = propagation.FrameTracer(sc, 1, cfg)
        tr.set_sources(w.sources[[s]], [s])
        t0 = time.time()
        d = dirs_of(w.seed, s, n)
        order = np.argsort(cell_key(d), kind="stable").astype(np.uint32)
        natural = np.arange(n, dtype=np.uint32)
        print(f"source {s}: host directions {time.time() - t0:.1f} s", flush=True)
        res = {}
        for name, ids in (("natural", natural), ("sorted", order), ("natural2", natural), ("sorted2", order)):
            ids_t = torch.as_tensor(ids.astype(np.int64)).to(torch.int32).cuda()
            for _ in range(2):
                tr.trace(w.listener, ray_ids=ids)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                tr.trace(w.listener, ray_ids=ids)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            segs = int(tr.stats[0, 1])
            res[name] = (ms, segs)
            print(f"  {name:9s} {ms:.3f} ms  {segs} segments  {segs / ms / 1e6:.3f} G seg/s", flush=True)


if __name__ == "__main__":
    main()
