"""Multi-GPU plumbing for the trace path.

Paths are independent, so rays shard by global index: of a frame of R rays
per source, rank g of N traces rays [g*R/N, (g+1)*R/N) of every source with
the same Philox streams as a single-GPU run (strong scaling: the frame is
fixed).  The only exchange is the per-frame histogram sum, so that each rank
ends up owning the complete histograms of S/N sources:

* fused (default): ef_trace_fused commits every splat straight into the
  owner's block over peer memory (PeerHistograms below);
* unfused: local partials (ef_trace) + one reduce-scatter -- torch's
  (reduce_scatter_sources; gloo for the CPU tests, which lacks
  reduce_scatter_tensor and falls back to all_reduce + slice) or the C ABI's
  ef_nccl_reduce_hist (NcclHistExchange).
"""
from __future__ import annotations

import ctypes


def shard_rays(rays_per_source: int, rank: int, world: int):
    """(ray0, n_rays) of this rank's slice of a frame of `rays_per_source`
    rays per source (strong scaling)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    if rays_per_source % world:
        raise ValueError(f"{rays_per_source} rays per source do not divide over {world} ranks")
    per = rays_per_source // world
    return rank * per, per


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


# --------------------------------------------------------------------------
# Fused trace + reduce-scatter over peer memory (ef_trace_fused)

class _CudaPeerBackend:
    """Device buffers through the C ABI: cudaMalloc + CUDA IPC handles."""

    def alloc(self, nbytes: int):
        import ctypes

        from . import _lib
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        _lib.check(_lib.lib().ef_peer_alloc(int(nbytes), ctypes.byref(p), h))
        return p.value, h.raw

    def open(self, handle: bytes):
        import ctypes

        from . import _lib
        p = ctypes.c_void_p()
        _lib.check(_lib.lib().ef_peer_open(ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(p)))
        return p.value

    def close(self, ptr):
        from . import _lib
        _lib.lib().ef_peer_close(ptr)

    def free(self, ptr):
        from . import _lib
        _lib.lib().ef_peer_free(ptr)

    def table(self, ptrs):
        import ctypes
        return (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])   # host array of device pointers

    def view(self, ptr, shape):
        from . import _lib
        return _lib.DeviceArray(ptr, shape).tensor()

    def sync(self):
        from . import _lib
        _lib.torch().cuda.current_stream().synchronize()


class PeerUnavailable(RuntimeError):
    """Peer-mapped histogram blocks could not be set up on every rank."""


class PeerHistograms:
    """This rank's share of the frame histograms, in peer-mapped memory.

    Rank r owns sources [r*S/N, (r+1)*S/N) (owned_sources).  Its histogram
    and direct-sound blocks are allocated here (ef_peer_alloc), the CUDA IPC
    handles are exchanged once (all_gather_object), and every rank maps every
    other rank's blocks (ef_peer_open) into two pointer tables (host arrays
    of device pointers, passed to the kernel by value).  The trace
    kernels of all ranks (FrameTracer.trace_fused -> ef_trace_fused) then add
    each splat straight into the owner's block over NVLink/NVSwitch: the
    reduce-scatter happens inside the trace, with no NCCL call after it.

    Double-buffered so that one barrier per frame orders everything: frame f
    accumulates into parity f & 1; ``begin_frame(f)`` zeroes this rank's
    parity (f+1) & 1 blocks for the next frame (after the owner consumed them
    two frames ago, stream order); ``end_frame()`` synchronises the stream and
    barriers, after which ``block(f)`` holds the complete sums of this rank's
    sources.  Both parities start zeroed."""

    def __init__(self, n_sources: int, n_bins: int, n_bands: int, nk: int, group=None,
                 backend=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        owned_sources(n_sources, self.rank, self.world)          # validates S % N == 0
        spr = n_sources // self.world
        self.sources_per_rank = spr
        self.shape_h = (spr, n_bins, n_bands, nk)
        self.shape_d = (spr, n_bands, nk)
        be = backend if backend is not None else _CudaPeerBackend()
        self._be = be
        nh = 4 * spr * n_bins * n_bands * nk
        nd = 4 * spr * n_bands * nk
        # Every rank takes part in every collective below even when a local
        # step fails, and the outcome is agreed on, so a rank that cannot map
        # its peers (no CUDA IPC / P2P) makes ALL ranks raise PeerUnavailable
        # together instead of leaving the others blocked in a collective.
        self._own, self._opened, self._tab = [], [], []
        err = None
        try:
            for _ in range(2):   # [(ptr, handle)] per parity
                self._own.append((be.alloc(nh), be.alloc(nd)))
            mine = [(h[1], d[1]) for h, d in self._own]
        except Exception as e:   # noqa: BLE001 - reported to every rank below
            err, mine = f"rank {self.rank}: peer allocation failed: {e}", None
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        if err is None and any(h is None for h in allh):
            err = "a peer could not allocate its blocks"
        if err is None:
            try:
                for parity in range(2):
                    hp, dp = [], []
                    for r in range(self.world):
                        if r == self.rank:
                            hp.append(self._own[parity][0][0])
                            dp.append(self._own[parity][1][0])
                        else:
                            ph = be.open(allh[r][parity][0])
                            self._opened.append(ph)
                            pd = be.open(allh[r][parity][1])
                            self._opened.append(pd)
                            hp.append(ph)
                            dp.append(pd)
                    self._tab.append((be.table(hp), be.table(dp)))
            except Exception as e:   # noqa: BLE001
                err = f"rank {self.rank}: mapping a peer's blocks failed: {e}"
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)
        bad = [x for x in errs if x]
        if bad:
            self._release()
            raise PeerUnavailable("; ".join(bad))
        self._H = [be.view(self._own[p][0][0], self.shape_h) for p in range(2)]
        self._D = [be.view(self._own[p][1][0], self.shape_d) for p in range(2)]

    def _release(self):
        for p in self._opened:
            self._be.close(p)
        for pair in self._own:
            for ptr, _ in pair:
                self._be.free(ptr)
        self._own, self._opened = None, []

    def tables(self, frame: int):
        """(hist table, dir table) pointer arrays (one device pointer per rank)
        for frame's parity."""
        return self._tab[frame & 1]

    def block(self, frame: int):
        """(H, Dir) of this rank's sources for `frame` (complete after end_frame)."""
        return self._H[frame & 1], self._D[frame & 1]

    def begin_frame(self, frame: int):
        nxt = (frame + 1) & 1
        self._H[nxt].zero_()
        self._D[nxt].zero_()

    def end_frame(self):
        import torch.distributed as dist

        self._be.sync()
        dist.barrier(group=self.group)

    def close(self):
        import torch.distributed as dist

        if self._own is None:
            return
        self._be.sync()
        dist.barrier(group=self.group)        # no peer still writes into our blocks
        self._release()


class EmulatedPeers:
    """N virtual ranks in one process and one GPU: every rank's blocks are
    local tensors and the pointer tables point at them, so ef_trace_fused
    runs exactly the addressing of the multi-GPU path (tests, 1-GPU boxes)."""

    def __init__(self, n_ranks: int, n_sources: int, n_bins: int, n_bands: int, nk: int):
        from . import _lib
        t = _lib.torch()
        dev = _lib.device()
        owned_sources(n_sources, 0, n_ranks)
        spr = n_sources // n_ranks
        self.world = n_ranks
        self.sources_per_rank = spr
        self._H = [[t.zeros((spr, n_bins, n_bands, nk), dtype=t.float32, device=dev)
                    for _ in range(n_ranks)] for _ in range(2)]
        self._D = [[t.zeros((spr, n_bands, nk), dtype=t.float32, device=dev)
                    for _ in range(n_ranks)] for _ in range(2)]
        import ctypes
        arr = ctypes.c_void_p * n_ranks
        self._tab = [(arr(*[x.data_ptr() for x in self._H[p]]), arr(*[x.data_ptr() for x in self._D[p]]))
                     for p in range(2)]

    def tables(self, frame: int):
        return self._tab[frame & 1]

    def block(self, frame: int, rank: int):
        return self._H[frame & 1][rank], self._D[frame & 1][rank]

    def begin_frame(self, frame: int):
        nxt = (frame + 1) & 1
        for x in self._H[nxt] + self._D[nxt]:
            x.zero_()

    def end_frame(self):
        pass


# --------------------------------------------------------------------------
# Unfused exchange through the C ABI's NCCL entry points (ef_nccl_*)
class NcclHistExchange:
    """ef_nccl_reduce_hist over a communicator made by ef_nccl_comm_create:
    rank 0's unique id travels over torch.distributed (any backend) when
    world > 1.  ``reduce_scatter(partial, owned)``: partial (S, ...) f32
    device tensor of this rank's ray shard, owned (S/N, ...) this rank's
    summed sources; ``all_reduce(buf)`` in place; ``reduce(buf)`` to rank 0."""

    def __init__(self, world: int | None = None, rank: int | None = None, device: int | None = None):
        from . import _lib
        t = _lib.torch()
        if world is None or rank is None:
            import torch.distributed as dist
            world, rank = dist.get_world_size(), dist.get_rank()
        self.world, self.rank = int(world), int(rank)
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _lib.check(_lib.lib().ef_nccl_unique_id(uid))
        if self.world > 1:
            import torch.distributed as dist
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0)
            ctypes.memmove(uid, box[0], 128)
        dev = t.cuda.current_device() if device is None else int(device)
        comm = ctypes.c_void_p()
        _lib.check(_lib.lib().ef_nccl_comm_create(self.world, self.rank, uid, dev, ctypes.byref(comm)))
        self._comm = comm

    def _run(self, partial, owned, count, mode, stream):
        from . import _lib
        t = _lib.torch()
        for x in (partial, owned):
            if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float32 and x.is_contiguous()):
                raise ValueError("NcclHistExchange: contiguous float32 CUDA tensors expected")
        _lib.check(_lib.lib().ef_nccl_reduce_hist(self._comm, _lib.ptr(partial), _lib.ptr(owned), count, mode,
                                                  _lib.stream_handle(stream)))

    def reduce_scatter(self, partial, owned, stream=None):
        if partial.shape[0] % self.world or owned.numel() * self.world != partial.numel():
            raise ValueError("NcclHistExchange.reduce_scatter: owned must hold 1/world of partial")
        self._run(partial, owned, owned.numel(), 0, stream)

    def all_reduce(self, buf, stream=None):
        self._run(buf, buf, buf.numel(), 1, stream)

    def reduce(self, buf, out=None, stream=None):
        out = buf if out is None else out
        self._run(buf, out, buf.numel(), 2, stream)

    def close(self):
        from . import _lib
        if getattr(self, "_comm", None) is not None and self._comm.value:
            _lib.check(_lib.lib().ef_nccl_comm_destroy(self._comm))
        self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
