"""ir-analysis on the B200.

``analyze`` runs the K4 decay-fit reducer (csrc/ef_analyze.cu) over every
(source, band) of a frame in one launch.  The SPEC's single-IR functions
(``estimate_rt60``, ``estimate_predelay``, ``average_directivity``) are thin
wrappers over the same kernel; ``reverb_gain`` / ``smooth_parameter`` are
closed forms.  Pinned estimator choices: DESIGN.md 3.6.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sh import SH_C0, n_coeffs
from .tdesigns import design_for_order

SILENT_RT60 = 1.0     # cold-start RT60 of a silent band


@dataclass
class ReverbParams:
    """Per-source analysis snapshot, numpy arrays."""
    rt60: np.ndarray              # (n_bands,) s
    reverb_gain: np.ndarray       # (n_bands,)
    drr_db: np.ndarray            # (n_bands,)
    total_intensity: np.ndarray   # (n_bands,)
    direct_intensity: np.ndarray  # (n_bands,)
    silent_bands: np.ndarray      # (n_bands,) bool
    predelay: float               # s, -1 when silent
    mean_free_path: float         # m
    avg_directivity: np.ndarray   # (n_bands, nk)
    loudness: np.ndarray | None   # (n_bands, nk, nk)
    silent: bool


class Analyzer:
    """Device output buffers for ef_analyze over (n_sources, n_bands)."""

    def __init__(self, n_sources: int, n_bins: int, n_bands: int, order: int,
                 bin_s: float, max_rt: float | None = None, loudness: bool = True):
        t = _lib.torch()
        dev = _lib.device()
        self.nk = n_coeffs(order)
        self.cfg = _lib.AnalysisConfig(n_sources, n_bins, n_bands, order, bin_s,
                                       max_rt if max_rt is not None else n_bins * bin_s)
        self.design = _lib.to_device(design_for_order(order).directions, t.float64)
        self.params = t.zeros((n_sources, n_bands, _lib.EF_P_COUNT), dtype=t.float64, device=dev)
        self.src_params = t.zeros((n_sources, _lib.EF_S_COUNT), dtype=t.float64, device=dev)
        self.avg_dir = t.zeros((n_sources, n_bands, self.nk), dtype=t.float64, device=dev)
        self.loudness = (t.zeros((n_sources, n_bands, self.nk, self.nk), dtype=t.float64, device=dev)
                         if loudness else None)

    def run(self, H, Dir, stats, sum_t, stream=None):
        _lib.check(_lib.lib().ef_analyze(
            self.cfg, _lib.ptr(H), _lib.ptr(Dir), _lib.ptr(stats), _lib.ptr(sum_t),
            _lib.ptr(self.design), self.design.shape[0], _lib.ptr(self.params),
            _lib.ptr(self.src_params), _lib.ptr(self.avg_dir), _lib.ptr(self.loudness),
            _lib.stream_handle(stream)))

    def results(self) -> list[ReverbParams]:
        p = self.params.cpu().numpy()
        q = self.src_params.cpu().numpy()
        a = self.avg_dir.cpu().numpy()
        d = self.loudness.cpu().numpy() if self.loudness is not None else None
        out = []
        for s in range(p.shape[0]):
            out.append(ReverbParams(
                rt60=p[s, :, 0], reverb_gain=p[s, :, 1], drr_db=p[s, :, 2],
                total_intensity=p[s, :, 3], direct_intensity=p[s, :, 4],
                silent_bands=p[s, :, 5] > 0.5, predelay=float(q[s, 0]),
                mean_free_path=float(q[s, 1]), avg_directivity=a[s],
                loudness=None if d is None else d[s], silent=bool(q[s, 2] > 0.5)))
        return out


def analyze(tracer, max_rt: float | None = None, loudness: bool = True) -> list[ReverbParams]:
    """Per-source ReverbParams of a FrameTracer's current histograms."""
    c = tracer.config
    an = Analyzer(tracer.n_sources, c.n_bins, tracer.nb, c.sh_order, c.bin_s,
                  max_rt if max_rt is not None else c.max_rt, loudness)
    an.run(tracer.H, tracer.Dir, tracer.stats, tracer.sum_t)
    return an.results()


def _single_band(ir_band, sample_rate, max_rt):
    """Run K4 on one intensity histogram (order 0, one band).  K4 reads f32
    histograms (the device accumulates in f32); the series is first scaled
    by a power of two (exact) that maps its maximum into [1, 2), so every
    non-zero bin stays non-zero in f32 unless it is below 2^-149 of the
    maximum (only estimate_predelay uses this path; RT60 takes the f64 one)."""
    t = _lib.torch()
    I = np.asarray(ir_band, dtype=np.float64).reshape(-1)
    peak = float(np.max(np.abs(I))) if I.size else 0.0
    if peak > 0.0 and np.isfinite(peak):
        I = I * 2.0 ** (-math.floor(math.log2(peak)))
    dev = _lib.device()
    H = t.as_tensor((I * SH_C0).astype(np.float32), device=dev).reshape(1, -1, 1, 1).contiguous()
    Dir = t.zeros((1, 1, 1), dtype=t.float32, device=dev)
    stats = t.zeros((1, _lib.EF_ST_COUNT), dtype=t.int64, device=dev)
    sum_t = t.zeros((1,), dtype=t.float64, device=dev)
    an = Analyzer(1, len(I), 1, 0, 1.0 / sample_rate, max_rt, loudness=False)
    an.run(H, Dir, stats, sum_t)
    return an.results()[0]


def estimate_rt60(ir_band, sample_rate: float = 100.0, max_rt: float = 8.0):
    """RT60 (s) of an intensity histogram, or None when silent/indeterminate
    (SPEC.md:272-280): Schroeder backward integration from the last non-zero
    bin, LS fit over -5..-35 dB (fallback -5..-25 dB), clamp [0.05, max_rt].
    The caller's f64 series goes to the device as f64: the same Schroeder fit
    as K4 (schroeder_fit, csrc/ef_analyze.cu) through ef_acoustic_metrics."""
    I = np.asarray(ir_band, dtype=np.float64).reshape(-1)
    if I.size == 0:
        return None
    rt = acoustic_metrics(I, 1.0 / sample_rate, max_rt=max_rt)["rt60"]
    return None if rt < 0 else float(rt)


def estimate_predelay(intensity, sample_rate: float = 100.0):
    """Time of the first bin with intensity > 0 in any band, None if silent
    (SPEC.md:299-307).  ``intensity``: (n_bins,) or (n_bins, n_bands)."""
    I = np.asarray(intensity, dtype=np.float64)
    if I.ndim == 1:
        I = I[:, None]
    firsts = []
    for b in range(I.shape[1]):
        r = _single_band(I[:, b], sample_rate, max(I.shape[0] / sample_rate, 0.05))
        if r.predelay >= 0:
            firsts.append(r.predelay)
    return min(firsts) if firsts else None


def reverb_gain(total_intensity: float, rt60: float) -> float:
    """g = sqrt(I_total / (RT60 / (6 ln 10)))."""
    if rt60 <= 0:
        raise ValueError("rt60 must be > 0")
    if total_intensity <= 0:
        return 0.0
    return math.sqrt(total_intensity / (rt60 / (6.0 * math.log(10.0))))


def smooth_parameter(new: float, cached: float, tau: float, dt: float) -> float:
    """a*new + (1-a)*cached, a = 1 - exp(-dt/tau)."""
    if tau <= 0 or dt <= 0:
        raise ValueError("tau and dt must be > 0")
    a = 1.0 - math.exp(-dt / tau)
    return a * new + (1.0 - a) * cached


def blend_histograms(cache, frame, alpha: float):
    """Device a*frame + (1-a)*cache (accumulate_ir)."""
    t = _lib.torch()
    if cache.shape != frame.shape:
        raise ValueError("histogram shapes differ")
    out = t.empty_like(frame)
    _lib.check(_lib.lib().ef_blend(_lib.ptr(cache.contiguous()), _lib.ptr(frame.contiguous()),
                                   frame.numel(), float(alpha), _lib.ptr(out), _lib.stream_handle()))
    return out


def blend_into(cache, frame, alpha: float):
    """In-place cache <- a*frame + (1-a)*cache on the device."""
    if cache.shape != frame.shape or not cache.is_contiguous() or not frame.is_contiguous():
        raise ValueError("cache and frame must be contiguous tensors of one shape")
    _lib.check(_lib.lib().ef_blend(_lib.ptr(cache), _lib.ptr(frame), frame.numel(), float(alpha),
                                   _lib.ptr(cache), _lib.stream_handle()))
    return cache


def acoustic_metrics(energy, bin_s: float, direct_index=0, e_ref: float = 1.0 / (4.0 * math.pi * 100.0),
                     max_rt: float = 8.0) -> dict:
    """RT60, C80, D50, TS, G per energy series on the
    device.  ``energy``: (n_bins,) or (n_bins, n_bands) energy per bin
    (pressure squared); metrics are measured from ``direct_index``; G is
    relative to ``e_ref`` (direct sound at 10 m in the free field)."""
    t = _lib.torch()
    E = np.asarray(energy, dtype=np.float64)
    single = E.ndim == 1
    E2 = np.ascontiguousarray((E[:, None] if single else E).T)          # (series, n_bins)
    dev = _lib.to_device(E2, t.float64)
    di = _lib.to_device(np.full(E2.shape[0], int(direct_index), np.int32), t.int32)
    out = t.zeros((E2.shape[0], 5), dtype=t.float64, device=dev.device)
    _lib.check(_lib.lib().ef_acoustic_metrics(_lib.ptr(dev), E2.shape[0], E2.shape[1], float(bin_s),
                                              _lib.ptr(di), float(e_ref), float(max_rt), _lib.ptr(out),
                                              _lib.stream_handle()))
    o = out.cpu().numpy()
    res = {k: o[:, i] for i, k in enumerate(("rt60", "c80", "d50", "ts", "g"))}
    return {k: float(v[0]) for k, v in res.items()} if single else res
