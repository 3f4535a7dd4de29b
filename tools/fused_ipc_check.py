"""Two-rank check of the fused trace over CUDA IPC (run under torchrun; both
ranks may share one GPU): each rank traces its ray shard of every source of
a small C3 interior (arrivals in every source block)
with ef_trace_fused into the owners' peer-mapped blocks; after end_frame its
own block must equal the unsharded frame of its sources (traced locally with
ef_trace).  gloo carries the handle exchange and the barriers."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import distributed, propagation, workloads  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    n_dev = torch.cuda.device_count()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % n_dev)
    w = workloads.c3_interior(n_sources=8, n_rays=2048)
    sc = scene_from_workload(w)
    S, R = len(w.sources), 1024
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    part = propagation.FrameTracer(sc, S, cfg)
    part.set_sources(w.sources)
    full = propagation.FrameTracer(sc, S, cfg)
    full.set_sources(w.sources)
    peers = distributed.PeerHistograms(S, w.n_bins, sc.n_bands, part.nk)
    spr = peers.sources_per_rank
    ok = True
    for frame in (0, 1, 2):
        peers.begin_frame(frame)
        part.trace_fused(w.listener, peers, frame=frame, ray0=rank * R, n_rays=R, total_rays=world * R)
        peers.end_frame()
        full.trace(w.listener, frame=frame, n_rays=world * R, total_rays=world * R)
        torch.cuda.synchronize()
        H, D = peers.block(frame)
        ref_h = full.H[rank * spr:(rank + 1) * spr]
        ref_d = full.Dir[rank * spr:(rank + 1) * spr]
        sc_h = float(ref_h.abs().max())
        nonzero = bool((H.flatten(1).abs().sum(1) > 0).all()) and sc_h > 0
        good = nonzero and (torch.allclose(H, ref_h, rtol=1e-5, atol=1e-6 * sc_h)
                and torch.allclose(D, ref_d, rtol=1e-5, atol=1e-6 * float(ref_d.abs().max())))
        if not good:
            print(f"rank {rank} frame {frame}: max |dH| {float((H - ref_h).abs().max()):.3e} "
                  f"of {sc_h:.3e}", flush=True)
        ok &= good
    peers.close()
    dist.destroy_process_group()
    if ok:
        print(f"fused-ipc ok rank {rank}", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
