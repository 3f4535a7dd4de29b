"""Propagation -- trace_frame and friends, on the B200.

The reference specifies this module but ships no code for it; the bounce
model is pinned in DESIGN.md section 3 (forward tracing from point sources to
a listener sphere, as BASELINE.json's configs require) and restated
independently in oracle/efo.c, which the parity tests compare against.

Hot path: one ``ef_trace`` launch traces every path of every source of a
frame inside one persistent kernel (no return to the host per bounce), and
commits arrivals straight into the device histogram
H[source, bin, band, sh] (float32).
"""
from __future__ import annotations

import ctypes

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .sh import SH_C0, n_coeffs

TAU_ER = 1.0
TAU_LR = 3.0


@dataclass
class TraceConfig:
    """Per-frame tracing parameters (SPEC RenderConfig subset, SPEC.md:589-592,
    extended with the BASELINE configs' receiver and histogram shape)."""
    primary_rays: int = 4096            # rays per source per frame
    max_order: int = 50                 # reflections per path
    sh_order: int = 2                   # histogram SH order (0..4)
    bin_s: float = 1e-3                 # IR bin width, s
    n_bins: int = 2000                  # IR length in bins
    listener_radius: float = 0.5        # m
    seed: int = 0
    mode: int = 0                       # 0 reference dispatch, 1 all-pairs, 2 BVH
    max_rt: float | None = None         # RT60 clamp (default: IR length)
    diffuse_rain: bool = False          # next-event connection per diffuse bounce
    er_max_order: int = 0               # arrivals of order 1..er_max_order -> PathList (<= 2)
    er_capacity: int = 1 << 20          # device ER list entries per launch

    @property
    def n_coeffs(self) -> int:
        return n_coeffs(self.sh_order)

    def e0(self, total_rays: int | None = None) -> float:
        """Initial per-band energy of a path: unit source power spread over
        the rays and normalised by the receiver cross-section."""
        n = self.primary_rays if total_rays is None else total_rays
        return float(np.float32(1.0 / (n * math.pi * self.listener_radius ** 2)))


@dataclass
class LowRateIR:
    """Energy IR with SH directivity.

    ``histogram[t, b, k]`` = sum over arrivals in bin t of E_b * Y_k(arrival);
    intensity = histogram[..., 0] / Y_00 and the directivity coefficients are
    histogram / intensity.  ``direct[b, k]`` holds order-0 (unreflected)
    arrivals.  Tensors stay on the device."""
    sample_rate: float
    histogram: object
    direct: object

    @property
    def length(self) -> int:
        return int(self.histogram.shape[0])

    @property
    def intensity(self):
        return self.histogram[..., 0] / SH_C0

    def numpy(self):
        return self.histogram.detach().cpu().numpy(), self.direct.detach().cpu().numpy()


@dataclass
class TraceStats:
    """SPEC.md:197-200 plus the receiver counters of DESIGN.md 3."""
    mean_free_path: float
    primary_rays_emitted: int
    total_segments: int
    reflections: int = 0
    arrivals: int = 0
    direct_arrivals: int = 0
    dropped_late: int = 0
    escaped: int = 0
    open_field: bool = False
    nodes_visited: int = 0        # device BVH work (not the reference's)
    triangles_tested: int = 0
    tail_segments: int = 0        # segments run by the frame-tail kernel


@dataclass
class PathList:
    """Early-reflection paths: one entry per distinct
    (source, reflection order, reflecting triangles) sequence of the frame's
    order <= er_max_order arrivals; delay = energy-weighted path length / c,
    pressure_b = sqrt(energy_b), directivity = energy-weighted order-2 SH of
    the arrival directions.  Empty unless enabled."""
    delays: np.ndarray = field(default_factory=lambda: np.zeros(0))
    pressures: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    directivities: np.ndarray = field(default_factory=lambda: np.zeros((0, 9)))
    kinds: list = field(default_factory=list)
    sources: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    orders: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    triangles: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.int64))
    dropped: int = 0

    def __len__(self) -> int:
        return len(self.delays)


def build_path_list(entries: np.ndarray, n_bands: int, speed_of_sound: float,
                    dropped: int = 0) -> PathList:
    """Group raw ER arrivals (ef_er_entry records) by reflection sequence."""
    from .sh import eval_sh_batch
    if len(entries) == 0:
        return PathList(pressures=np.zeros((0, n_bands)), dropped=dropped)
    key = np.stack([entries["src"], entries["order"], entries["tri0"], entries["tri1"]], 1)
    uniq, inv = np.unique(key, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    e = entries["energy"][:, :n_bands].astype(np.float64)
    etot = e.sum(1)
    g = len(uniq)
    esum = np.zeros((g, n_bands))
    np.add.at(esum, inv, e)
    wsum = np.bincount(inv, weights=etot, minlength=g)
    dist = np.bincount(inv, weights=etot * entries["dist"], minlength=g) / np.maximum(wsum, 1e-300)
    Y = eval_sh_batch(entries["dir"].astype(np.float64), 2)
    ysum = np.zeros((g, 9))
    np.add.at(ysum, inv, Y * etot[:, None])
    return PathList(delays=dist / speed_of_sound, pressures=np.sqrt(esum),
                    directivities=ysum / np.maximum(wsum, 1e-300)[:, None],
                    kinds=["early-reflection"] * g, sources=uniq[:, 0].astype(np.int64),
                    orders=uniq[:, 1].astype(np.int64), triangles=uniq[:, 2:].astype(np.int64),
                    dropped=dropped)


@dataclass
class CoherenceCaches:
    """Temporal coherence caches.

    * ``ir``: per source key, the exponentially smoothed LowRateIR
      (accumulate_ir, tau_LR = 3 s).
    * ``er``: the diffuse path cache -- per reflection sequence (source,
      order, first two triangles), exponentially smoothed per-band energies,
      SH directivity and delay (tau_ER = 1 s).  A sequence missing from a
      frame decays with the same blend (its frame contribution is zero).
    * entries not refreshed for 2 tau expire (``clock`` is the time of the
      latest update)."""
    tau_lr: float = TAU_LR
    tau_er: float = TAU_ER
    ir: dict = field(default_factory=dict)
    er: dict = field(default_factory=dict)
    ir_seen: dict = field(default_factory=dict)
    clock: float = 0.0

    def update_er(self, paths: "PathList", dt: float) -> "PathList":
        """Fold one frame's PathList into the diffuse path cache; returns the
        cached paths (ER go to the PathList via this cache)."""
        if dt <= 0:
            raise ValueError("dt must be > 0")
        self.clock += dt
        a = 1.0 - math.exp(-dt / self.tau_er) if self.tau_er > 0 else 1.0
        fresh = {}
        for j in range(len(paths)):
            k = (int(paths.sources[j]), int(paths.orders[j]), int(paths.triangles[j][0]),
                 int(paths.triangles[j][1]))
            fresh[k] = (paths.pressures[j] ** 2, paths.directivities[j], float(paths.delays[j]))
        nb = paths.pressures.shape[1] if len(paths) else (
            next(iter(self.er.values()))["energy"].shape[0] if self.er else 4)
        for k in set(self.er) | set(fresh):
            e_new, y_new, d_new = fresh.get(k, (np.zeros(nb), np.zeros(9), None))
            c = self.er.get(k)
            if c is None:
                self.er[k] = {"energy": np.array(e_new, float), "dir": np.array(y_new, float),
                              "delay": d_new, "seen": self.clock}
                continue
            c["energy"] = a * np.asarray(e_new, float) + (1.0 - a) * c["energy"]
            c["dir"] = a * np.asarray(y_new, float) + (1.0 - a) * c["dir"]
            if d_new is not None:
                c["delay"] = d_new
                c["seen"] = self.clock
        self.expire()
        keys = sorted(self.er)
        if not keys:
            return PathList(pressures=np.zeros((0, nb)), dropped=paths.dropped)
        E = np.stack([self.er[k]["energy"] for k in keys])
        return PathList(delays=np.array([self.er[k]["delay"] for k in keys]),
                        pressures=np.sqrt(E), directivities=np.stack([self.er[k]["dir"] for k in keys]),
                        kinds=["early-reflection"] * len(keys),
                        sources=np.array([k[0] for k in keys], np.int64),
                        orders=np.array([k[1] for k in keys], np.int64),
                        triangles=np.array([[k[2], k[3]] for k in keys], np.int64),
                        dropped=paths.dropped)

    def touch_ir(self, key):
        self.ir_seen[key] = self.clock

    def expire(self):
        """Drop entries not refreshed for 2 tau."""
        for k in [k for k, c in self.er.items() if self.clock - c["seen"] > 2.0 * self.tau_er]:
            del self.er[k]
        for k in [k for k, t in self.ir_seen.items() if self.clock - t > 2.0 * self.tau_lr]:
            self.ir.pop(k, None)
            del self.ir_seen[k]


def _stats_from_row(row: np.ndarray, sum_t: float) -> TraceStats:
    paths, segs, refl, arr, direct, dropped, esc, nodes, tris, tail = (int(x) for x in row[:10])
    return TraceStats(mean_free_path=sum_t / refl if refl else 0.0,
                      primary_rays_emitted=paths, total_segments=segs, reflections=refl,
                      arrivals=arr, direct_arrivals=direct, dropped_late=dropped, escaped=esc,
                      open_field=refl == 0, nodes_visited=nodes, triangles_tested=tris,
                      tail_segments=tail)


class FrameTracer:
    """Device buffers + launches for repeated frames over a fixed scene and
    source count: the batched form of ``trace_frame`` used by the bench and
    the multi-source configs.  ``trace()`` is one ef_trace launch (plus a
    histogram clear); nothing synchronises the host."""

    def __init__(self, scene, n_sources: int, config: TraceConfig, record: bool = False):
        t = _lib.torch()
        dev = _lib.device()
        self.scene = scene
        self.config = config
        self.n_sources = n_sources
        self.nb = scene.n_bands
        self.nk = config.n_coeffs
        # H | Dir | stats | sum_t in one allocation, in that order: ef_trace
        # then clears a frame's outputs with one memset instead of four
        nh = n_sources * config.n_bins * self.nb * self.nk
        nd = n_sources * self.nb * self.nk
        o_st = -(-4 * (nh + nd) // 8) * 8
        o_su = o_st + 8 * n_sources * _lib.EF_ST_COUNT
        self._outputs = t.zeros(o_su + 8 * n_sources, dtype=t.uint8, device=dev)
        buf = self._outputs
        self.H = buf[:4 * nh].view(t.float32).view(n_sources, config.n_bins, self.nb, self.nk)
        self.Dir = buf[4 * nh:4 * (nh + nd)].view(t.float32).view(n_sources, self.nb, self.nk)
        self.stats = buf[o_st:o_su].view(t.int64).view(n_sources, _lib.EF_ST_COUNT)
        self.sum_t = buf[o_su:].view(t.float64)
        self.src_pos = t.zeros((n_sources, 3), dtype=t.float64, device=dev)
        self.src_key = t.arange(n_sources, dtype=t.int32, device=dev)
        self.record = record
        self.path_nseg = None
        self.path_ids = None
        self.er = None
        self.er_count = None
        if config.er_max_order > 0:
            self.er = t.zeros((config.er_capacity * _lib.ER_DTYPE.itemsize,), dtype=t.uint8, device=dev)
            self.er_count = t.zeros((1,), dtype=t.int32, device=dev)
        self._handle = scene._device_handle()

    def set_sources(self, positions, keys=None):
        t = _lib.torch()
        self.src_pos.copy_(t.as_tensor(np.asarray(positions, np.float64).reshape(-1, 3)))
        if keys is not None:
            self.src_key.copy_(t.as_tensor(np.asarray(keys, np.int64).astype(np.int32)))

    def clear(self):
        self.H.zero_()
        self.Dir.zero_()
        self.stats.zero_()
        self.sum_t.zero_()

    def _launch_config(self, listener, frame, ray0, n_rays, total_rays, ray_ids, clear):
        t = _lib.torch()
        c = self.config
        ids = None
        if ray_ids is not None:
            ids = _lib.to_device(np.asarray(ray_ids, np.uint32).astype(np.int64), t.int64).to(t.int32)
            n_rays = ids.shape[0]
        n_rays = c.primary_rays if n_rays is None else int(n_rays)
        cfg = _lib.TraceConfig()
        cfg.n_sources = self.n_sources
        cfg.order = c.sh_order
        cfg.n_bins = c.n_bins
        cfg.max_bounces = c.max_order
        cfg.n_rays = n_rays
        cfg.ray0 = ray0
        cfg.seed = c.seed & 0xffffffff
        cfg.frame = frame & 0xffffffff
        cfg.mode = c.mode
        cfg.bin_len = self.scene.speed_of_sound * c.bin_s
        lp = np.asarray(listener, np.float64).reshape(3)
        cfg.listener[:] = [float(x) for x in lp]
        cfg.radius = c.listener_radius
        cfg.e0 = c.e0(total_rays)
        cfg.record_ids = int(self.record)
        cfg.clear_outputs = int(bool(clear))
        cfg.diffuse_rain = int(bool(c.diffuse_rain))
        if self.er is not None:
            if clear:
                self.er_count.zero_()
            cfg.er_max_order = min(int(c.er_max_order), 2)
            cfg.er_capacity = int(c.er_capacity)
            cfg.er_entries = self.er.data_ptr()
            cfg.er_count = self.er_count.data_ptr()
        self.path_nseg = self.path_ids = None
        if self.record:
            self.path_nseg = t.zeros((self.n_sources, n_rays), dtype=t.int32, device=self.H.device)
            self.path_ids = t.full((self.n_sources, n_rays, c.max_order), -2, dtype=t.int32,
                                   device=self.H.device)
        return cfg, ids

    def trace(self, listener, frame: int = 0, ray0: int = 0, n_rays: int | None = None,
              total_rays: int | None = None, ray_ids=None, clear: bool = True, stream=None):
        """Launch ef_trace for all sources (rays [ray0, ray0+n_rays) of each,
        or the explicit global indices ``ray_ids``)."""
        cfg, ids = self._launch_config(listener, frame, ray0, n_rays, total_rays, ray_ids, clear)
        _lib.check(_lib.lib().ef_trace(
            self._handle, cfg, _lib.ptr(self.src_pos), _lib.ptr(self.src_key), _lib.ptr(ids),
            _lib.ptr(self.H), _lib.ptr(self.Dir), _lib.ptr(self.stats), _lib.ptr(self.sum_t),
            _lib.ptr(self.path_nseg), _lib.ptr(self.path_ids), _lib.stream_handle(stream)))

    def trace_fused(self, listener, peers, frame: int = 0, ray0: int = 0, n_rays: int | None = None,
                    total_rays: int | None = None, ray_ids=None, stream=None, slot: int | None = None):
        """Multi-GPU frame slice through ef_trace_fused: the splats of every
        source go straight into its owner's block of ``peers``
        (distributed.PeerHistograms, buffer ``slot`` -- the frame sequence
        number given to begin_frame, default ``frame``), so no reduce-scatter
        follows.  Stats / sum_t / ER stay local to this tracer."""
        cfg, ids = self._launch_config(listener, frame, ray0, n_rays, total_rays, ray_ids, True)
        tab_h, tab_d = peers.tables(frame if slot is None else slot)
        _lib.check(_lib.lib().ef_trace_fused(
            self._handle, cfg, _lib.ptr(self.src_pos), _lib.ptr(self.src_key), _lib.ptr(ids),
            ctypes.cast(tab_h, ctypes.c_void_p), ctypes.cast(tab_d, ctypes.c_void_p),
            peers.sources_per_rank, _lib.ptr(self.stats),
            _lib.ptr(self.sum_t), _lib.ptr(self.path_nseg), _lib.ptr(self.path_ids),
            _lib.stream_handle(stream)))

    def early_reflections(self) -> np.ndarray:
        """Raw ER arrivals of the last trace (structured ef_er_entry array)."""
        if self.er is None:
            return np.zeros(0, _lib.ER_DTYPE)
        n = min(int(self.er_count.item()), self.config.er_capacity)
        return self.er[:n * _lib.ER_DTYPE.itemsize].cpu().numpy().view(_lib.ER_DTYPE).copy()

    def path_list(self) -> PathList:
        n_total = 0 if self.er is None else int(self.er_count.item())
        raw = self.early_reflections()
        return build_path_list(raw, self.nb, self.scene.speed_of_sound,
                               dropped=max(0, n_total - self.config.er_capacity))

    def irs(self):
        return [LowRateIR(1.0 / self.config.bin_s, self.H[s], self.Dir[s]) for s in range(self.n_sources)]

    def trace_stats(self):
        st = self.stats.cpu().numpy()
        sm = self.sum_t.cpu().numpy()
        return [_stats_from_row(st[s], float(sm[s])) for s in range(self.n_sources)]


def trace_frame(scene, source, listener, config: TraceConfig, caches: CoherenceCaches | None = None,
                rng=None, frame: int = 0, dt: float | None = None):
    """Trace one frame for one source.

    ``rng``: an int seed (overrides config.seed) or None.  Returns
    (PathList, LowRateIR, TraceStats).  With ``caches`` and ``dt`` the IR is
    folded into the temporal IR cache (accumulate_ir) and the early
    reflections into the diffuse path cache, and the cached versions are
    returned."""
    if config.primary_rays < 1 or config.max_order < 1:
        raise ValueError("config.primary_rays and config.max_order must be >= 1")
    seed = config.seed if rng is None else int(rng)
    cfg = TraceConfig(**{**config.__dict__, "seed": seed})
    pos = source.pose_at(frame * (dt or 0.0)) if hasattr(source, "pose_at") else np.asarray(source)
    lpos = listener.pose_at(frame * (dt or 0.0))[0] if hasattr(listener, "pose_at") else np.asarray(listener)
    # the source's index in the scene keys its RNG stream and its IR cache
    # entry (by identity: positions are arrays, so == is elementwise)
    key = next((i for i, s in enumerate(getattr(scene, "sources", [])) if s is source), 0)
    if scene.n_triangles == 0:
        t = _lib.torch()
        dev = _lib.device()
        ir = LowRateIR(1.0 / cfg.bin_s, t.zeros((cfg.n_bins, scene.n_bands, cfg.n_coeffs), device=dev),
                       t.zeros((scene.n_bands, cfg.n_coeffs), device=dev))
        return PathList(), ir, TraceStats(0.0, cfg.primary_rays, cfg.primary_rays, open_field=True)
    tr = FrameTracer(scene, 1, cfg)
    tr.set_sources(np.asarray(pos)[None, :], [key])
    tr.trace(lpos, frame=frame)
    ir = tr.irs()[0]
    paths = tr.path_list() if cfg.er_max_order > 0 else PathList()
    if caches is not None and dt is not None:
        # advance the clock and expire first, so an entry older than 2 tau is
        # dropped rather than blended into this frame's IR; then blend, store
        # and mark the entry fresh (the returned IR is the cached one)
        if cfg.er_max_order > 0:
            paths = caches.update_er(paths, dt)      # advances the clock, expires ER and IR
        else:
            caches.clock += dt
            caches.expire()
        ir = accumulate_ir(caches.ir.get(key), ir, caches.tau_lr, dt)
        caches.ir[key] = ir
        caches.touch_ir(key)
    return paths, ir, tr.trace_stats()[0]


def accumulate_ir(cache_ir: LowRateIR | None, frame_ir: LowRateIR, tau: float, dt: float) -> LowRateIR:
    """out = a*frame + (1-a)*cache, a = 1 - exp(-dt/tau)."""
    if dt <= 0:
        raise ValueError("dt must be > 0")
    if cache_ir is None:
        return frame_ir
    a = 1.0 - math.exp(-dt / tau) if tau > 0 else 1.0
    from .analysis import blend_histograms
    return LowRateIR(frame_ir.sample_rate,
                     blend_histograms(cache_ir.histogram, frame_ir.histogram, a),
                     blend_histograms(cache_ir.direct, frame_ir.direct, a))


def compute_direct_sound(scene, source, listener, rng=None, samples: int = 64, order: int = 3,
                         power: float = 1.0, t: float = 0.0) -> PathList:
    """Direct path entry.  Point source (radius 0): one
    visibility ray; intensity P/(4 pi d^2), directivity Y(direction to the
    source).  Spherical source: `samples` directions uniform in the cone it
    subtends, each tested for visibility (ef_occluded_batch); the entry
    carries the visible fraction of the intensity and the mean SH projection
    of the visible directions.  A fully occluded source yields pressure 0."""
    from .sh import eval_sh_batch
    sp = np.asarray(source.pose_at(t) if hasattr(source, "pose_at") else source, np.float64)
    lp = np.asarray(listener.pose_at(t)[0] if hasattr(listener, "pose_at") else listener, np.float64)
    radius = float(getattr(source, "radius", 0.0))
    gain = float(getattr(source, "gain", 1.0))
    v = sp - lp
    dist = float(np.linalg.norm(v))
    if dist <= 0.0:
        raise ValueError("source and listener coincide")
    axis = v / dist
    intensity = power * gain * gain / (4.0 * np.pi * dist * dist)
    nb = scene.n_bands
    if radius <= 0.0 or radius >= dist:
        dirs = axis[None, :]
        targets = sp[None, :]
    else:
        rng = np.random.default_rng(rng)
        cos_max = np.sqrt(1.0 - (radius / dist) ** 2)
        z = rng.uniform(cos_max, 1.0, samples)
        phi = rng.uniform(0.0, 2.0 * np.pi, samples)
        r = np.sqrt(1.0 - z * z)
        # orthonormal basis around the axis (Duff et al.)
        sg = np.copysign(1.0, axis[2])
        a = -1.0 / (sg + axis[2])
        b = axis[0] * axis[1] * a
        t1 = np.array([1.0 + sg * axis[0] * axis[0] * a, sg * b, -sg * axis[0]])
        t2 = np.array([b, sg + axis[1] * axis[1] * a, -axis[1]])
        dirs = (r * np.cos(phi))[:, None] * t1 + (r * np.sin(phi))[:, None] * t2 + z[:, None] * axis
        # target: where the direction meets the source sphere (near side)
        tc = dirs @ v
        disc = np.maximum(tc * tc - (dist * dist - radius * radius), 0.0)
        targets = lp + (tc - np.sqrt(disc))[:, None] * dirs
    blocked = scene.occluded_batch(np.repeat(lp[None, :], len(dirs), axis=0), targets)
    vis = ~np.asarray(blocked)
    frac = float(vis.mean())
    Y = eval_sh_batch(dirs[vis], order).mean(axis=0) if vis.any() else np.zeros((order + 1) ** 2)
    p = np.sqrt(intensity * frac)
    return PathList(delays=np.array([dist / scene.speed_of_sound]), pressures=np.full((1, nb), p),
                    directivities=Y[None, :], kinds=["direct"], sources=np.array([0]),
                    orders=np.array([0]), triangles=np.full((1, 2), -1))
