"""SH-domain auralization on the B200 (BASELINE config C4).

``SHRenderer(params)`` uploads per-source parameters once; ``process(x)``
renders one 512-sample block for every source: LR4 crossover into band
histories, direct tap + order-3 SH encode, a 16-line FDN per band fed at the
predelay, lines -> SH through g_reverb,b * D_b * E, and the overlap-save
binaural decode of the 16-channel bus -- 2(n+1)^2 = 32 convolutions per
block regardless of the source count.  Semantics: DESIGN.md
3.7; CPU restatement: oracle/audio.py.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

FS = 48000.0
BLOCK = 512
N_LINES = 16
EDGES = (176.0, 775.0, 3408.0)


class AudioConfig(ctypes.Structure):
    _fields_ = [("n_sources", ctypes.c_int32), ("hist_len", ctypes.c_int32),
                ("line_len", ctypes.c_int32), ("reserved", ctypes.c_int32)]


def _biquad(kind, f0, q=1.0 / np.sqrt(2.0)):
    w0 = 2.0 * np.pi * f0 / FS
    c, s = np.cos(w0), np.sin(w0)
    al = s / (2.0 * q)
    b = {"lp": [(1 - c) / 2, 1 - c, (1 - c) / 2], "hp": [(1 + c) / 2, -(1 + c), (1 + c) / 2],
         "ap": [1 - al, -2 * c, 1 + al]}[kind]
    a0, a1, a2 = 1 + al, -2 * c, 1 - al
    return [b[0] / a0, b[1] / a0, b[2] / a0, a1 / a0, a2 / a0]


def crossover_sos() -> np.ndarray:
    """(4 bands, 5 biquads, [b0 b1 b2 a1 a2]): LR4 tree at 176/775/3408 Hz
    with allpass compensation so the band sum is allpass."""
    f1, f2, f3 = EDGES
    lr = lambda k, f: [_biquad(k, f), _biquad(k, f)]  # noqa: E731
    return np.array([lr("lp", f2) + lr("lp", f1) + [_biquad("ap", f3)],
                     lr("lp", f2) + lr("hp", f1) + [_biquad("ap", f3)],
                     lr("hp", f2) + lr("lp", f3) + [_biquad("ap", f1)],
                     lr("hp", f2) + lr("hp", f3) + [_biquad("ap", f1)]], dtype=np.float32)


def line_directions() -> np.ndarray:
    i = np.arange(N_LINES)
    z = 1.0 - (2.0 * i + 1.0) / N_LINES
    r = np.sqrt(1.0 - z * z)
    phi = i * np.pi * (3.0 - np.sqrt(5.0))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def _split_delay(D):
    D = np.asarray(D, np.float64)
    fl = np.floor(D)
    return fl.astype(np.int32), (1.0 - (D - fl)).astype(np.float32)


def _per_source(p: dict, m: np.ndarray) -> dict:
    """The per-source device arrays of a parameter set (line delays m fixed):
    direct SH encoding, split direct delay / predelay, direct gains, FDN line
    gains 10^(-3 m_i / (fs RT60_b)) (Eq. 7) and the line -> SH matrices
    g_reverb,b * D_b * E."""
    from .sh import eval_sh_batch
    Y = eval_sh_batch(p["dir_direct"], 3).astype(np.float32)
    E = eval_sh_batch(line_directions(), 3).T * np.sqrt(4.0 * np.pi / N_LINES)   # (16 sh, 16 lines)
    g_line = (10.0 ** (-3.0 * m[:, None, :].astype(np.float64) / (FS * p["rt60"][:, :, None])))
    M = p["g_reverb"][:, :, None, None] * np.einsum("sbkj,ji->sbki", p["D"], E)
    d_int, d_w = _split_delay(p["delay_direct"])
    p_int, p_w = _split_delay(p["predelay"])
    arrs = dict(Y=Y, d_int=d_int, d_w=d_w, gain=np.asarray(p["gain_direct"], np.float32), p_int=p_int,
                p_w=p_w, g=g_line.astype(np.float32), M=M.astype(np.float32))
    return {k: np.ascontiguousarray(v) for k, v in arrs.items()}


class SHRenderer:
    """Device state + launches of ef_audio_* for S sources."""

    def __init__(self, params: dict, hist_len: int | None = None, line_len: int = 4096):
        p = params
        S = p["dir_direct"].shape[0]
        self.S = S
        m = p["fdn_delay"].astype(np.int32)
        self._m = m
        H = np.fft.rfft(np.concatenate([p["hrtf"], np.zeros(p["hrtf"].shape[:2] + (1024 - p["hrtf"].shape[2],))],
                                       axis=2), axis=2).astype(np.complex64)
        src = _per_source(p, m)
        d_int, p_int = src["d_int"], src["p_int"]
        if hist_len is None:
            # smallest power-of-two band history holding the longest tap + a block
            need = int(max(d_int.max(), p_int.max())) + BLOCK + 2
            hist_len = 1 << max(need - 1, 1).bit_length()
        self.hist_len = hist_len
        arrs = dict(sos=crossover_sos(), m=m, H=np.ascontiguousarray(H).view(np.float32), **src)
        self._host = {k: np.ascontiguousarray(v) for k, v in arrs.items()}
        cfg = AudioConfig(S, hist_len, line_len, 0)
        h = ctypes.c_void_p()
        a = self._host
        _lib.check(_lib.lib().ef_audio_create(
            ctypes.byref(cfg), *[_lib.host_ptr(a[k]) for k in
                                 ("sos", "Y", "d_int", "d_w", "gain", "p_int", "p_w", "m", "g", "M", "H")],
            ctypes.byref(h)))
        self._h = h
        t = _lib.torch()
        dev = _lib.device()
        self.bus = t.zeros((16, BLOCK), dtype=t.float32, device=dev)
        self.out = t.zeros((2, BLOCK), dtype=t.float32, device=dev)

    def update_params(self, params: dict, stream=None) -> None:
        """update_params: swap direct encoding / delay /
        gains, predelay, RT60-derived line gains and g_reverb * D at the next
        block boundary (blocks already enqueued on the stream keep the old
        values).  The FDN line delays and the HRTF stay those of creation;
        the band histories, line rings and filter states carry over."""
        if np.asarray(params["dir_direct"]).shape[0] != self.S:
            raise ValueError("update_params: source count differs from the renderer's")
        a = _per_source(params, self._m)
        _lib.check(_lib.lib().ef_audio_update(
            self._h, *[_lib.host_ptr(a[k]) for k in ("Y", "d_int", "d_w", "gain", "p_int", "p_w", "g", "M")],
            _lib.stream_handle(stream)))
        self._host.update(a)

    def device_bytes(self) -> int:
        o = np.zeros(4, np.int64)
        _lib.check(_lib.lib().ef_audio_info(self._h, _lib.host_ptr(o)))
        return int(o[1])

    def process(self, x, want_bus: bool = True, stream=None):
        """x: (S, 512) f32 (numpy or CUDA tensor) -> (bus (16,512), out (2,512))."""
        t = _lib.torch()
        is_np = not (isinstance(x, t.Tensor) and x.is_cuda)
        xd = _lib.to_device(x, t.float32, (self.S, BLOCK))
        _lib.check(_lib.lib().ef_audio_process(self._h, _lib.ptr(xd),
                                               _lib.ptr(self.bus) if want_bus else None,
                                               _lib.ptr(self.out), _lib.stream_handle(stream)))
        if is_np:
            return self.bus.cpu().numpy(), self.out.cpu().numpy()
        return self.bus, self.out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.ef_audio_destroy(h)
            self._h = None


def params_from_estimates(estimates, sources, listener, fdn_delay, hrtf, speed_of_sound: float = 343.0,
                          band_groups=None, fallback_rt60: float = 1.0) -> dict:
    """C4 renderer parameters from the estimator's per-source ReverbParams
    (analysis.Analyzer.results(); BASELINE configs[3]: "reverb send using
    estimated parameters").  The renderer has 4 bands (LR4 at 176/775/3408
    Hz); an estimate with N_b bands is folded onto them in contiguous groups
    (``band_groups``, default N_b/4 bands each: C3's 8 bands pairwise):
    RT60 = mean over the group (silent bands: ``fallback_rt60``),
    g_reverb = rms, D = mean of the directional loudness matrices, direct
    gain = sqrt(mean direct intensity) (pressure of the direct path).
    Direct direction / delay come from the geometry (listener -> source), the
    predelay from the estimate (the direct delay when silent).  ``fdn_delay``
    (S, 16) samples and ``hrtf`` (16, 2, taps) are the renderer's own."""
    S = len(estimates)
    nb = len(estimates[0].rt60)
    if band_groups is None:
        if nb % 4:
            raise ValueError("params_from_estimates: give band_groups for a band count not divisible by 4")
        k = nb // 4
        band_groups = [list(range(i * k, (i + 1) * k)) for i in range(4)]
    src = np.asarray(sources, np.float64).reshape(S, 3)
    v = src - np.asarray(listener, np.float64).reshape(1, 3)
    dist = np.linalg.norm(v, axis=1)
    if np.any(dist <= 0.0):
        raise ValueError("params_from_estimates: a source coincides with the listener")
    rt60 = np.zeros((S, 4))
    g_rev = np.zeros((S, 4))
    gain = np.zeros((S, 4))
    D = np.zeros((S, 4, 16, 16))
    pre = np.zeros(S)
    delay = dist / speed_of_sound * FS
    for s, e in enumerate(estimates):
        if e.loudness is None or e.loudness.shape[-1] != 16:
            raise ValueError("params_from_estimates: needs order-3 loudness matrices")
        for b, grp in enumerate(band_groups):
            r = np.where(e.silent_bands[grp], fallback_rt60, e.rt60[grp])
            rt60[s, b] = float(np.mean(r))
            g_rev[s, b] = float(np.sqrt(np.mean(np.asarray(e.reverb_gain[grp]) ** 2)))
            gain[s, b] = float(np.sqrt(max(np.mean(e.direct_intensity[grp]), 0.0)))
            D[s, b] = np.mean(e.loudness[grp], axis=0)
        pre[s] = e.predelay * FS if e.predelay >= 0 else delay[s]
    return dict(dir_direct=v / dist[:, None], delay_direct=delay, gain_direct=gain, predelay=pre,
                fdn_delay=np.asarray(fdn_delay, np.int32), rt60=rt60, g_reverb=g_rev, D=D,
                hrtf=np.asarray(hrtf))


THRESHOLD_OF_HEARING = 1e-12   # W/m^2
N_ER = 100                     # rendered early reflections (§5)


def prioritize_paths(paths, threshold: float = THRESHOLD_OF_HEARING, max_paths: int = N_ER):
    """render_early's path selection: drop paths whose
    intensity (sum over bands of pressure^2) is below the threshold of
    hearing, sort the rest by decreasing intensity (stable: equal intensities
    keep their order) and keep the first ``max_paths`` across all sources.
    Returns (kept PathList, dropped PathList) -- the dropped reflection paths
    go back to the IR for reinjection."""
    from .propagation import PathList
    P = np.asarray(paths.pressures, np.float64)
    inten = (P ** 2).sum(axis=1) if len(paths) else np.zeros(0)
    audible = np.nonzero(inten >= threshold)[0]
    order = audible[np.argsort(-inten[audible], kind="stable")]
    keep, drop = order[:max_paths], np.setdiff1d(np.arange(len(paths)), order[:max_paths])

    def take(idx):
        return PathList(delays=np.asarray(paths.delays)[idx], pressures=P[idx],
                        directivities=np.asarray(paths.directivities)[idx],
                        kinds=[paths.kinds[i] for i in idx],
                        sources=np.asarray(paths.sources)[idx] if len(paths.sources) else paths.sources,
                        orders=np.asarray(paths.orders)[idx] if len(paths.orders) else paths.orders,
                        triangles=np.asarray(paths.triangles)[idx] if len(paths.triangles) else paths.triangles)
    kept, dropped = take(keep), take(drop)
    kept.dropped = len(drop)
    return kept, dropped
