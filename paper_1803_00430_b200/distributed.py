"""Multi-GPU plumbing for the trace path.

Paths are independent, so rays shard by global index: rank g traces rays
[g*R, (g+1)*R) of every source with the same Philox streams as a single-GPU
run.  The only exchange is the per-frame histogram sum, done with one
reduce-scatter over the source axis so that each rank ends up owning the
complete histograms of S/N sources (NCCL over NVLink on the B200 box; gloo
for the CPU tests, which lacks reduce_scatter_tensor and falls back to
all_reduce + slice).
"""
from __future__ import annotations


def shard_rays(rays_per_rank: int, rank: int):
    """(ray0, n_rays) of this rank's slice (weak scaling: fixed per rank)."""
    return rank * rays_per_rank, rays_per_rank


def owned_sources(n_sources: int, rank: int, world: int):
    if n_sources % world:
        raise ValueError(f"{n_sources} sources do not divide over {world} ranks")
    per = n_sources // world
    return slice(rank * per, (rank + 1) * per)


def reduce_scatter_sources(full, group=None):
    """Sum `full` (sources leading) over ranks; return this rank's S/N block."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sl = owned_sources(full.shape[0], rank, world)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((full.shape[0] // world,) + tuple(full.shape[1:]), dtype=full.dtype,
                          device=full.device)
        dist.reduce_scatter_tensor(out, full.contiguous(), group=group)
        return out
    buf = full.clone()
    dist.all_reduce(buf, group=group)
    return buf[sl].contiguous()
