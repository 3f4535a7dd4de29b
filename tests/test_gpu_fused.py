"""Fused trace + reduce-scatter (ef_trace_fused, distributed.PeerHistograms).

* N virtual ranks in one process (EmulatedPeers): every rank traces its ray
  shard of all sources and its splats land in the owners' blocks through the
  pointer tables; each owner block equals the unsharded single-GPU frame.
* Two processes on the one GPU (CUDA IPC, gloo barriers): the real peer
  mapping.  The two trace kernels never wait on each other (host barriers
  only), so sharing a GPU is safe.
Run on a B200 with ``-m gpu``."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1803_00430_b200 import distributed, propagation, workloads  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tracer(w, sc, n_src):
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius,
                                  seed=w.seed)
    tr = propagation.FrameTracer(sc, n_src, cfg)
    tr.set_sources(w.sources[:n_src])
    return tr


def _close(a, b):
    """Equal up to f32 atomic ordering -- and never a zero-vs-zero pass."""
    scale = float(b.abs().max())
    assert scale > 0 and float(a.abs().max()) > 0, "vacuous comparison: empty block"
    return torch.allclose(a, b, rtol=1e-5, atol=1e-6 * scale)


_C3 = {}


def _c3():
    """C3 interior (closed room: ~2 arrivals per 1,000 segments), 8 sources
    of 1,024 rays per rank: every owner block of every rank gets splats."""
    if not _C3:
        w = workloads.c3_interior(n_sources=8, n_rays=4096)
        _C3["w"], _C3["sc"] = w, scene_from_workload(w)
    return _C3["w"], _C3["sc"]


@pytest.mark.parametrize("ranks", [2, 4])
def test_fused_emulated_ranks_equal_unsharded(ranks):
    """Each rank traces rays [r*R, (r+1)*R) of every source with
    ef_trace_fused into the owners' blocks; every owner block (non-zero)
    equals the unsharded frame of its sources, and equals what the unfused
    exchange (per-rank ef_trace partials + a reduce-scatter, summed here as
    NCCL would) delivers to that owner."""
    w, sc = _c3()
    S, R = len(w.sources), 1024
    full = _tracer(w, sc, S)
    part = _tracer(w, sc, S)
    peers = distributed.EmulatedPeers(ranks, S, w.n_bins, sc.n_bands, full.nk)
    spr = S // ranks
    for frame in (0, 1, 2):
        full.trace(w.listener, frame=frame, n_rays=ranks * R, total_rays=ranks * R)
        peers.begin_frame(frame)
        segs = 0
        partial_h, partial_d = [], []
        for r in range(ranks):
            part.trace_fused(w.listener, peers, frame=frame, ray0=r * R, n_rays=R,
                             total_rays=ranks * R)
            segs += int(part.stats[:, 1].sum())
        peers.end_frame()
        for r in range(ranks):       # the unfused form: local partials of every source
            part.trace(w.listener, frame=frame, ray0=r * R, n_rays=R, total_rays=ranks * R)
            partial_h.append(part.H.clone())
            partial_d.append(part.Dir.clone())
        torch.cuda.synchronize()
        assert int(full.stats[:, 3].min()) > 0          # every source has arrivals
        rs_h = torch.stack(partial_h).sum(0)             # reduce-scatter: owner r gets rows r*spr..
        rs_d = torch.stack(partial_d).sum(0)
        for r in range(ranks):
            H, D = peers.block(frame, r)
            own = slice(r * spr, (r + 1) * spr)
            assert _close(H, full.H[own]) and _close(D, full.Dir[own])
            assert _close(H, rs_h[own]) and _close(D, rs_d[own])
            for j in range(spr):                          # every owned source block is non-zero
                assert float(H[j].abs().sum()) > 0
        assert segs == int(full.stats[:, 1].sum())


def test_fused_two_processes_over_cuda_ipc():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "fused_ipc_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count("fused-ipc ok") == 2, r.stdout[-2000:]
