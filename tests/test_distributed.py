"""Multi-rank path on CPU (gloo, world size 2): ray shards traced by the
oracle on each rank and reduce-scattered with the product's helper equal the
unsharded frame (counts exactly, histograms to f64 rounding)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_frame(w, src_ids, ray0, n):
    from oracle import oracle as O
    os_ = O.OracleScene.from_arrays(w.arrays())
    H, stats = [], []
    for s in src_ids:
        r = O.trace(os_, src_key=s, src_pos=w.sources[s], listener=w.listener, radius=w.radius,
                    seed=w.seed, order=w.order, n_bins=w.n_bins, bin_len=w.speed_of_sound * w.bin_s,
                    max_bounces=w.max_bounces, e0=1.0, ray0=ray0, n_rays=n)
        H.append(r.H)
        stats.append([r.stats["segments"], r.stats["arrivals"], r.stats["reflections"]])
    return np.array(H), np.array(stats, dtype=np.float64)


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1803_00430_b200 import distributed, workloads
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = workloads.c1_shoebox()
    w.sources = np.array([[2.0, 2.0, 1.5], [3.0, 6.0, 1.0]])
    ray0, nr = distributed.shard_rays(world * n, rank, world)
    H, st = _oracle_frame(w, [0, 1], ray0, nr)
    Hr = distributed.reduce_scatter_sources(torch.from_numpy(H))
    Sr = distributed.reduce_scatter_sources(torch.from_numpy(st))
    q.put((rank, Hr.numpy(), Sr.numpy()))
    dist.destroy_process_group()


def test_sharded_frame_equals_unsharded():
    from paper_1803_00430_b200 import workloads
    world, n = 2, 512
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (h, s)) for r, h, s in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = workloads.c1_shoebox()
    w.sources = np.array([[2.0, 2.0, 1.5], [3.0, 6.0, 1.0]])
    H, st = _oracle_frame(w, [0, 1], 0, world * n)
    for r in range(world):
        h, s = res[r]
        assert np.array_equal(s[0], st[r])                     # exact counts
        np.testing.assert_allclose(h[0], H[r], rtol=1e-12, atol=1e-18)


def test_owned_sources_validation():
    from paper_1803_00430_b200 import distributed
    assert distributed.owned_sources(8, 1, 4) == slice(2, 4)
    with pytest.raises(ValueError):
        distributed.owned_sources(7, 0, 2)


# ---------------------------------------------------------------- fused path
class _ShmBackend:
    """CPU stand-in for the CUDA IPC backend of distributed.PeerHistograms:
    buffers are files in shared memory, a handle is the file name, opening a
    handle maps the same pages (what cudaIpcOpenMemHandle does for device
    memory)."""

    def __init__(self, tmpdir, rank):
        self.tmpdir, self.rank, self.maps, self.k = tmpdir, rank, {}, 0

    def _map(self, path):
        self.k += 1
        self.maps[self.k] = np.memmap(path, np.float32, "r+")
        return self.k

    def alloc(self, nbytes):
        path = os.path.join(self.tmpdir, f"r{self.rank}_{self.k}")
        np.memmap(path, np.float32, "w+", shape=(nbytes // 4,)).flush()
        return self._map(path), path.encode().ljust(64, b"\0")

    def open(self, handle):
        return self._map(bytes(handle).rstrip(b"\0").decode())

    def close(self, p):
        self.maps.pop(p)

    free = close

    def table(self, ptrs):
        return list(ptrs)

    def view(self, p, shape):
        return torch.from_numpy(self.maps[p]).view(shape)

    def sync(self):
        for m in self.maps.values():
            m.flush()


def _fused_worker(rank, world, port, n, tmpdir, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1803_00430_b200 import distributed, workloads
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = workloads.c1_shoebox()
    w.sources = np.array([[2.0, 2.0, 1.5], [3.0, 6.0, 1.0], [5.0, 3.0, 2.0], [1.0, 7.0, 1.2]])
    S = len(w.sources)
    be = _ShmBackend(tmpdir, rank)
    peers = distributed.PeerHistograms(S, w.n_bins, w.absorption.shape[1], (w.order + 1) ** 2,
                                       backend=be)
    assert peers.sources_per_rank == S // world
    out = []
    for frame in (0, 1, 2):
        peers.begin_frame(frame)
        tab_h, _ = peers.tables(frame)
        ray0, nr = distributed.shard_rays(world * n, rank, world)
        from oracle import oracle as O
        os_ = O.OracleScene.from_arrays(w.arrays())
        for turn in range(world):                       # one writer at a time (no CPU atomics)
            if turn == rank:
                for g in range(S):
                    r = O.trace(os_, src_key=g, src_pos=w.sources[g], listener=w.listener,
                                radius=w.radius, seed=w.seed, frame=frame, order=w.order,
                                n_bins=w.n_bins, bin_len=w.speed_of_sound * w.bin_s,
                                max_bounces=w.max_bounces, e0=1.0, ray0=ray0, n_rays=nr)
                    o = g // peers.sources_per_rank
                    blk = be.maps[tab_h[o]].reshape(peers.shape_h)
                    blk[g % peers.sources_per_rank] += r.H.astype(np.float32)
                be.sync()
            dist.barrier()
        peers.end_frame()
        out.append(peers.block(frame)[0].numpy().copy())
    peers.close()
    q.put((rank, out))
    dist.destroy_process_group()


def test_peer_histograms_protocol(tmp_path):
    """distributed.PeerHistograms on world size 2 over gloo with a shared-
    memory backend: handles exchanged and mapped per rank, splats routed to
    the owner's block through the pointer tables, double-buffered frames --
    after end_frame each rank's block equals the unsharded frame of its
    sources, for three consecutive frames."""
    from oracle import oracle as O
    from paper_1803_00430_b200 import workloads
    world, n = 2, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, n, str(tmp_path), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = workloads.c1_shoebox()
    w.sources = np.array([[2.0, 2.0, 1.5], [3.0, 6.0, 1.0], [5.0, 3.0, 2.0], [1.0, 7.0, 1.2]])
    os_ = O.OracleScene.from_arrays(w.arrays())
    for frame in (0, 1, 2):
        for g in range(len(w.sources)):
            r = O.trace(os_, src_key=g, src_pos=w.sources[g], listener=w.listener, radius=w.radius,
                        seed=w.seed, frame=frame, order=w.order, n_bins=w.n_bins,
                        bin_len=w.speed_of_sound * w.bin_s, max_bounces=w.max_bounces, e0=1.0,
                        ray0=0, n_rays=world * n)
            blk = res[g // 2][frame][g % 2]
            scale = np.abs(r.H).max()
            np.testing.assert_allclose(blk, r.H, rtol=1e-5, atol=1e-6 * scale)


class _FailingOpenBackend(_ShmBackend):
    """Rank 1 cannot map its peer's blocks (no IPC / P2P on this node)."""

    def open(self, handle):
        if self.rank == 1:
            raise OSError("cudaIpcOpenMemHandle: peer access not supported")
        return super().open(handle)


def _unavailable_worker(rank, world, port, tmpdir, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1803_00430_b200 import distributed
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        distributed.PeerHistograms(4, 16, 4, 16, backend=_FailingOpenBackend(tmpdir, rank))
        q.put((rank, "no error"))
    except distributed.PeerUnavailable as e:
        q.put((rank, "unavailable: " + str(e)))
    dist.barrier()                 # both ranks got here: nobody hangs in a collective
    dist.destroy_process_group()


def test_peer_setup_failure_is_agreed_by_every_rank(tmp_path):
    """One rank failing to map its peers makes every rank raise
    PeerUnavailable (bench.py then falls back to the NCCL exchange), instead
    of leaving the others blocked in a collective."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_unavailable_worker, args=(r, world, port, str(tmp_path), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(v.startswith("unavailable") and "rank 1" in v for v in res.values()), res
