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
    scale = float(b.abs().max())
    return torch.allclose(a, b, rtol=1e-5, atol=1e-6 * scale)


@pytest.mark.parametrize("ranks", [2, 4])
def test_fused_emulated_ranks_equal_unsharded(ranks):
    w = workloads.c2_city()
    sc = scene_from_workload(w)
    S, R = len(w.sources), 2048
    full = _tracer(w, sc, S)
    part = _tracer(w, sc, S)
    peers = distributed.EmulatedPeers(ranks, S, w.n_bins, sc.n_bands, full.nk)
    for frame in (0, 1, 2):
        full.trace(w.listener, frame=frame, n_rays=ranks * R)
        peers.begin_frame(frame)
        segs = 0
        for r in range(ranks):
            part.trace_fused(w.listener, peers, frame=frame, ray0=r * R, n_rays=R,
                             total_rays=ranks * R)
            segs += int(part.stats[:, 1].sum())
        peers.end_frame()
        torch.cuda.synchronize()
        spr = S // ranks
        for r in range(ranks):
            H, D = peers.block(frame, r)
            assert _close(H, full.H[r * spr:(r + 1) * spr])
            assert _close(D, full.Dir[r * spr:(r + 1) * spr])
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
