"""C4 driven by estimates, and the unfused NCCL exchange through the C ABI.
Run on a B200 with ``-m gpu``.

* A C3 frame (8 bands, order 3) is traced and K4 estimates RT60 / gain /
  DRR / loudness / predelay per source; ``render.params_from_estimates`` maps
  them onto C4's 4-band renderer, and ``SHRenderer.update_params`` swaps them
  in at a block boundary.  Device vs the f64 oracle (same
  swap at the same boundary): error <= -80 dB relative to signal.
* ``ef_nccl_reduce_hist``: a one-rank communicator over the
  real libnccl -- reduce-scatter / all-reduce / reduce of ef_trace partials
  equal their sum."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1803_00430_b200 import _lib, analysis, distributed, propagation, render, workloads  # noqa: E402
from paper_1803_00430_b200.scene import scene_from_workload  # noqa: E402


def _err_db(a, ref):
    return 10 * np.log10(np.sum((a - ref) ** 2) / max(np.sum(ref ** 2), 1e-300))


def test_c4_renderer_driven_by_c3_estimates():
    from oracle import audio as OA4
    w = workloads.c3_interior(n_sources=4, n_rays=4096)
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, 4, cfg)
    tr.set_sources(w.source_positions(0))
    tr.trace(w.listener)
    est = analysis.analyze(tr)
    assert all(not e.silent_bands.all() for e in est)
    p0 = workloads.c4_params(n_sources=4)
    p1 = render.params_from_estimates(est, w.source_positions(0), w.listener, p0["fdn_delay"], p0["hrtf"])
    assert np.all(p1["rt60"] > 0.05) and np.all(p1["g_reverb"] > 0) and np.all(p1["predelay"] > 0)
    # the estimates differ from the synthetic start: the swap is observable
    assert np.abs(p1["rt60"] - p0["rt60"]).max() > 0.05
    x = workloads.pink_noise(4, 16 * 512)
    r = render.SHRenderer(p0, hist_len=8192)
    ora = OA4.AudioOracle(p0, p0["hrtf"])
    bus_g, out_g, bus_o, out_o = [], [], [], []
    for k in range(16):
        if k == 6:   # block boundary: swap to the estimated parameters
            r.update_params(p1)
            ora.update(p1)
        blk = x[:, k * 512:(k + 1) * 512]
        b, o = r.process(blk)
        bo, oo = ora.process(blk)
        bus_g.append(b.copy()); out_g.append(o.copy()); bus_o.append(bo); out_o.append(oo)
    bus_g, bus_o = np.concatenate(bus_g, 1), np.concatenate(bus_o, 1)
    out_g, out_o = np.concatenate(out_g, 1), np.concatenate(out_o, 1)
    assert np.abs(out_o[:, 6 * 512:]).max() > 0
    assert _err_db(bus_g, bus_o) <= -80.0, _err_db(bus_g, bus_o)
    assert _err_db(out_g, out_o) <= -80.0, _err_db(out_g, out_o)
    # without the swap the oracle's output differs: the update took effect
    ora2 = OA4.AudioOracle(p0, p0["hrtf"])
    out2 = np.concatenate([ora2.process(x[:, k * 512:(k + 1) * 512])[1] for k in range(16)], 1)
    assert _err_db(out2[:, 8 * 512:], out_o[:, 8 * 512:]) > -40.0


def test_update_params_rejects_bad_delays():
    p0 = workloads.c4_params(n_sources=2)
    r = render.SHRenderer(p0)
    bad = dict(p0)
    bad["predelay"] = np.full(2, 1e6)
    with pytest.raises(ValueError):
        r.update_params(bad)


def test_nccl_reduce_hist_one_rank():
    ex = distributed.NcclHistExchange(world=1, rank=0)
    w = workloads.c3_interior(n_sources=2, n_rays=1024)
    sc = scene_from_workload(w)
    cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                  bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = propagation.FrameTracer(sc, 2, cfg)
    tr.set_sources(w.sources)
    tr.trace(w.listener)
    owned = torch.empty_like(tr.H)
    ex.reduce_scatter(tr.H, owned)
    torch.cuda.synchronize()
    assert float(tr.H.abs().sum()) > 0 and torch.equal(owned, tr.H)
    acc = tr.H.clone()
    ex.all_reduce(acc)
    torch.cuda.synchronize()
    assert torch.equal(acc, tr.H)
    with pytest.raises(ValueError):
        ex.reduce_scatter(tr.H, owned[:1])
    ex.close()
