"""Freeze the algorithmic work per segment of the REFERENCE algorithm
(SURVEY.md 8(d)): BVH nodes visited and triangles tested by bvh.py:130-160
(brute force, 12 triangles, for C1), and the listener-arrival fraction, by
running the CPU oracle's instrumented copy on real segments of a config.

    python tools/measure_work.py c2 [rays_per_source]

Output feeds DESIGN.md section 5 and bench.py's B_SEG table."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1803_00430_b200 import workloads  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    w = workloads.WORKLOADS[name]()
    n = int(sys.argv[2]) if len(sys.argv) > 2 else w.n_rays
    n_src = int(sys.argv[3]) if len(sys.argv) > 3 else len(w.sources)
    t0 = time.time()
    os_ = O.OracleScene.from_arrays(w.arrays())
    build = time.time() - t0
    tot = dict.fromkeys(O.ST_NAMES, 0)
    t0 = time.time()
    for s in range(n_src):
        r = O.trace(os_, src_key=s, src_pos=w.sources[s], listener=w.listener, radius=w.radius,
                    seed=w.seed, order=w.order, n_bins=w.n_bins, bin_len=w.speed_of_sound * w.bin_s,
                    max_bounces=w.max_bounces, e0=1.0, n_rays=n)
        for k, v in r.stats.items():
            tot[k] += v
    dt = time.time() - t0
    seg = tot["segments"]
    nb, nk = w.n_bands, (w.order + 1) ** 2
    n_node = tot["nodes"] / seg
    n_tri = tot["tris"] / seg
    p_arr = tot["arrivals"] / seg
    b_seg = 72 * n_tri + 32 * n_node + (28 + 8 * nb) + p_arr * 8 * nb * nk
    print(json.dumps(dict(config=name, n_tri_scene=w.n_tri, rays_per_source=n,
                          sources=n_src, seg_per_path=seg / tot["paths"],
                          N_node=round(n_node, 3), N_tri=round(n_tri, 3), P_arr=p_arr,
                          B_seg=round(b_seg, 1), oracle_build_s=round(build, 2),
                          oracle_seg_per_s_1thread=round(seg / dt), **tot)))


if __name__ == "__main__":
    main()
