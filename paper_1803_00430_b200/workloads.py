"""Seeded synthetic workloads with the shapes of BASELINE.json configs C1-C5.

The paper's benchmark scenes (City, Hospital, ...) are not
shipped with the reference (pkg/.gitignore excludes /examples/), so every
config is a seeded stand-in with the named sizes and value distributions
(SURVEY.md section 8(d)).  Every box uses the 12-triangle face order of
``make_box_scene`` (scene.py:363-370) so triangle ids are predictable.

Geometry is produced as the reference's triangle soup: ``v0 = A``,
``e1 = B - A``, ``e2 = C - A`` (scene.py:325).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# corner index = 4*ix + 2*iy + iz (ix,iy,iz in {0: lo, 1: hi}); two triangles
# per face in the order -x, +x, -y, +y, -z, +z (scene.py:360-370)
_BOX_FACES = np.array([
    [0, 1, 3], [0, 3, 2],
    [4, 6, 7], [4, 7, 5],
    [0, 4, 5], [0, 5, 1],
    [2, 3, 7], [2, 7, 6],
    [0, 2, 6], [0, 6, 4],
    [1, 5, 7], [1, 7, 3],
], dtype=np.int64)


def box_triangles(lo, hi):
    """(12,3,3) triangles of the axis-aligned box [lo, hi]."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    corners = np.array([[(lo, hi)[ix][0], (lo, hi)[iy][1], (lo, hi)[iz][2]]
                        for ix in (0, 1) for iy in (0, 1) for iz in (0, 1)])
    return corners[_BOX_FACES]


def _rng(cfg: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([cfg, stream]))


@dataclass
class Workload:
    name: str
    tris: np.ndarray              # (T,3,3) float64 vertices A,B,C
    material_index: np.ndarray    # (T,) int64
    absorption: np.ndarray        # (M, n_bands)
    scattering: np.ndarray        # (M, n_bands)
    sources: np.ndarray           # (S,3) positions (frame 0)
    listener: np.ndarray          # (3,)
    radius: float
    n_rays: int                   # rays per source per frame
    max_bounces: int
    order: int
    n_bins: int = 2000
    bin_s: float = 1e-3
    seed: int = 0
    n_frames: int = 1
    frame_dt: float = 0.0
    source_velocity: np.ndarray | None = None   # (S,3) m/s
    speed_of_sound: float = 343.0
    notes: dict = field(default_factory=dict)

    @property
    def n_bands(self) -> int:
        return self.absorption.shape[1]

    @property
    def n_tri(self) -> int:
        return len(self.tris)

    def soup(self):
        A, B, C = self.tris[:, 0], self.tris[:, 1], self.tris[:, 2]
        return (np.ascontiguousarray(A), np.ascontiguousarray(B - A),
                np.ascontiguousarray(C - A))

    def normals(self):
        """Unit normals exactly as SceneModel.__init__ (scene.py:163-166)."""
        _, e1, e2 = self.soup()
        cross = np.cross(e1, e2)
        return cross / np.linalg.norm(cross, axis=1)[:, None]

    def source_positions(self, frame: int) -> np.ndarray:
        if self.source_velocity is None:
            return self.sources
        return self.sources + self.source_velocity * (frame * self.frame_dt)

    def arrays(self) -> dict:
        v0, e1, e2 = self.soup()
        return dict(v0=v0, e1=e1, e2=e2, normals=self.normals(),
                    material_index=self.material_index,
                    absorption=self.absorption, scattering=self.scattering)


def c1_shoebox() -> Workload:
    """C1: 10x8x3 m shoebox, 12 triangles, one material per wall."""
    tris = box_triangles((0.0, 0.0, 0.0), (10.0, 8.0, 3.0))
    mat = np.repeat(np.arange(6, dtype=np.int64), 2)
    absorption = _rng(1, 0).uniform(0.05, 0.4, size=(6, 4))
    scattering = np.full((6, 4), 0.5)
    return Workload("c1_shoebox", tris, mat, absorption, scattering,
                    sources=np.array([[2.0, 2.0, 1.5]]), listener=np.array([7.0, 5.0, 1.5]),
                    radius=0.5, n_rays=4096, max_bounces=50, order=2, seed=0)


def _street_points(rng, n, lo, hi, footprints, margin, z):
    pts = []
    while len(pts) < n:
        p = rng.uniform(lo, hi, size=2)
        inside = ((p[0] > footprints[:, 0] - margin) & (p[0] < footprints[:, 2] + margin) &
                  (p[1] > footprints[:, 1] - margin) & (p[1] < footprints[:, 3] + margin))
        if not inside.any():
            pts.append([p[0], p[1], z])
    return np.array(pts)


def c2_city(n_boxes: int = 200, n_sources: int = 8, n_rays: int = 32768) -> Workload:
    """C2: 500x500 m ground + 200 boxes (footprint U[5,30], height U[5,60])."""
    rng = _rng(2, 0)
    ground = np.array([[[0, 0, 0], [500, 0, 0], [500, 500, 0]],
                       [[0, 0, 0], [500, 500, 0], [0, 500, 0]]], dtype=np.float64)
    w = rng.uniform(5, 30, size=(n_boxes, 2))
    h = rng.uniform(5, 60, size=n_boxes)
    x = rng.uniform(0, 500 - w[:, 0])
    y = rng.uniform(0, 500 - w[:, 1])
    boxes = [box_triangles((x[i], y[i], 0.0), (x[i] + w[i, 0], y[i] + w[i, 1], h[i]))
             for i in range(n_boxes)]
    tris = np.concatenate([ground] + boxes)
    mat = np.concatenate([np.zeros(2, np.int64), np.repeat(np.arange(1, n_boxes + 1), 12)])
    absorption = _rng(2, 1).uniform(0.02, 0.3, size=(n_boxes + 1, 4))
    scattering = np.full((n_boxes + 1, 4), 0.5)
    foot = np.stack([x, y, x + w[:, 0], y + w[:, 1]], axis=1)
    pts = _street_points(_rng(2, 2), n_sources + 1, 0.0, 500.0, foot, 1.0, 1.5)
    return Workload("c2_city", tris, mat, absorption, scattering, sources=pts[:n_sources],
                    listener=pts[n_sources], radius=0.5, n_rays=n_rays, max_bounces=100,
                    order=3, seed=2)


def _box_surface_grid(lo, hi, cells, jitter, rng):
    """Closed, shared-vertex subdivided surface of box [lo,hi] (watertight):
    vertices on an integer lattice of the surface, jittered once each."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    n = np.asarray(cells)
    jit = {}

    def vert(ix, iy, iz):
        key = (ix, iy, iz)
        if key not in jit:
            jit[key] = rng.normal(0.0, jitter, size=3)
        base = lo + (hi - lo) * np.array([ix, iy, iz]) / n
        return base + jit[key]

    tris = []
    for axis in range(3):
        a1, a2 = [a for a in range(3) if a != axis]
        for side in (0, n[axis]):
            for i in range(n[a1]):
                for j in range(n[a2]):
                    q = []
                    for di, dj in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        idx = [0, 0, 0]
                        idx[axis] = side
                        idx[a1] = i + di
                        idx[a2] = j + dj
                        q.append(vert(*idx))
                    tris.append([q[0], q[1], q[2]])
                    tris.append([q[0], q[2], q[3]])
    return np.array(tris)


def c3_interior(cells=(130, 130, 26), n_boxes: int = 400, n_sources: int = 32,
                n_rays: int = 65536, n_frames: int = 64) -> Workload:
    """C3: 20x20x4 m room, jittered subdivided walls + 400 boxes (~100k tris),
    8 bands, 32 sources moving at 1-2 m/s over 64 frames of 16.7 ms."""
    rng = _rng(3, 0)
    room = _box_surface_grid((0, 0, 0), (20, 20, 4), cells, 0.01, rng)
    fw = rng.uniform(0.3, 1.5, size=(n_boxes, 2))
    fh = rng.uniform(0.3, 1.2, size=n_boxes)
    fx = rng.uniform(0.5, 19.5 - fw[:, 0])
    fy = rng.uniform(0.5, 19.5 - fw[:, 1])
    boxes = [box_triangles((fx[i], fy[i], 0.0), (fx[i] + fw[i, 0], fy[i] + fw[i, 1], fh[i]))
             for i in range(n_boxes)]
    tris = np.concatenate([room] + boxes)
    mat = np.concatenate([np.zeros(len(room), np.int64),
                          np.repeat(np.arange(1, n_boxes + 1), 12)])
    absorption = _rng(3, 1).uniform(0.02, 0.3, size=(n_boxes + 1, 8))
    scattering = np.full((n_boxes + 1, 8), 0.5)
    srng = _rng(3, 2)
    src = srng.uniform([3, 3, 1.5], [17, 17, 1.5], size=(n_sources, 3))
    ang = srng.uniform(0, 2 * np.pi, size=n_sources)
    spd = srng.uniform(1.0, 2.0, size=n_sources)
    vel = np.stack([np.cos(ang) * spd, np.sin(ang) * spd, np.zeros(n_sources)], axis=1)
    return Workload("c3_interior", tris, mat, absorption, scattering, sources=src,
                    listener=np.array([10.0, 10.0, 1.7]), radius=0.5, n_rays=n_rays,
                    max_bounces=64, order=3, seed=3, n_frames=n_frames, frame_dt=0.0167,
                    source_velocity=vel)


def _subdivided_box(lo, hi, nh, nv):
    """Walls split into nh x nv quads each plus a 2-triangle roof (no floor)."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    out = []
    zs = np.linspace(lo[2], hi[2], nv + 1)
    for axis, side in ((0, 0), (0, 1), (1, 0), (1, 1)):
        other = 1 - axis
        fixed = (lo, hi)[side][axis]
        ts = np.linspace(lo[other], hi[other], nh + 1)
        for i in range(nh):
            for j in range(nv):
                def p(t, z):
                    v = np.zeros(3)
                    v[axis] = fixed
                    v[other] = t
                    v[2] = z
                    return v
                a, b, c, d = p(ts[i], zs[j]), p(ts[i + 1], zs[j]), p(ts[i + 1], zs[j + 1]), p(ts[i], zs[j + 1])
                out.append([a, b, c])
                out.append([a, c, d])
    roof = box_triangles(lo, hi)[10:12]
    return np.concatenate([np.array(out), roof])


def c5_city_grid(nx: int = 50, ny: int = 40, nh: int = 6, nv: int = 10,
                 n_sources: int = 256, n_rays: int = 1 << 20) -> Workload:
    """C5: ground + 2,000 boxes on a grid with subdivided facades (~964k tris)."""
    rng = _rng(5, 0)
    pitch = 40.0
    ext = np.array([nx * pitch, ny * pitch])
    ground = np.array([[[0, 0, 0], [ext[0], 0, 0], [ext[0], ext[1], 0]],
                       [[0, 0, 0], [ext[0], ext[1], 0], [0, ext[1], 0]]], dtype=np.float64)
    w = rng.uniform(15, 30, size=(nx * ny, 2))
    h = rng.uniform(8, 80, size=nx * ny)
    boxes = []
    foot = []
    for k in range(nx * ny):
        gx, gy = k % nx, k // nx
        x0 = gx * pitch + (pitch - w[k, 0]) / 2
        y0 = gy * pitch + (pitch - w[k, 1]) / 2
        boxes.append(_subdivided_box((x0, y0, 0.0), (x0 + w[k, 0], y0 + w[k, 1], h[k]), nh, nv))
        foot.append([x0, y0, x0 + w[k, 0], y0 + w[k, 1]])
    per = len(boxes[0])
    tris = np.concatenate([ground] + boxes)
    mat = np.concatenate([np.zeros(2, np.int64), np.repeat(np.arange(1, nx * ny + 1), per)])
    absorption = _rng(5, 1).uniform(0.02, 0.3, size=(nx * ny + 1, 8))
    scattering = np.full((nx * ny + 1, 8), 0.5)
    pts = _street_points(_rng(5, 2), n_sources + 1, 0.0, float(ext.min()), np.array(foot), 1.0, 1.5)
    return Workload("c5_city_grid", tris, mat, absorption, scattering, sources=pts[:n_sources],
                    listener=pts[n_sources], radius=0.5, n_rays=n_rays, max_bounces=100,
                    order=3, seed=5)


WORKLOADS = {"c1": c1_shoebox, "c2": c2_city, "c3": c3_interior, "c5": c5_city_grid}


def _sh3_np(d):
    """Order-3 real SH (sh.py:94-115 formulas) for synthetic-parameter
    generation only; the render path uses the device eval_sh."""
    d = np.asarray(d, np.float64).reshape(-1, 3)
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    xx, yy, zz = x * x, y * y, z * z
    return np.stack([
        np.full_like(x, 0.28209479177387814), -0.4886025119029199 * y, 0.4886025119029199 * z,
        -0.4886025119029199 * x, 1.0925484305920792 * x * y, -1.0925484305920792 * y * z,
        0.31539156525252005 * (2.0 * zz - xx - yy), -1.0925484305920792 * x * z,
        0.5462742152960396 * (xx - yy), -0.5900435899266435 * y * (3.0 * xx - yy),
        2.890611442640554 * x * y * z, -0.4570457994644658 * y * (4.0 * zz - xx - yy),
        0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
        -0.4570457994644658 * x * (4.0 * zz - xx - yy), 1.445305721320277 * z * (xx - yy),
        -0.5900435899266435 * x * (xx - 3.0 * yy)], axis=1)


def pink_noise(n_sources: int, n_samples: int, seed: int = 4) -> np.ndarray:
    """Seeded pink noise (Kellet's three-pole filter on white noise), f32."""
    rng = _rng(seed, 7)
    w = rng.standard_normal((n_sources, n_samples))
    out = np.zeros_like(w)
    b0 = np.zeros(n_sources)
    b1 = np.zeros(n_sources)
    b2 = np.zeros(n_sources)
    for i in range(n_samples):
        wi = w[:, i]
        b0 = 0.99765 * b0 + wi * 0.0990460
        b1 = 0.96300 * b1 + wi * 0.2965164
        b2 = 0.57000 * b2 + wi * 1.0526913
        out[:, i] = b0 + b1 + b2 + wi * 0.1848
    return (0.1 * out).astype(np.float32)


def c4_params(n_sources: int = 64, seed: int = 4) -> dict:
    """C4: per-source estimated parameters (C1/C2-like ranges), FDN delays
    ~U[20, 80] ms, and 16x2 seeded exponentially decaying 256-tap filters."""
    rng = _rng(seed, 0)
    S = n_sources
    d = rng.standard_normal((S, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    dist = rng.uniform(2.0, 30.0, size=S)
    fs = 48000.0
    rt60 = rng.uniform(0.4, 1.5, size=(S, 4))
    total = rng.uniform(0.005, 0.05, size=(S, 4))
    g_reverb = np.sqrt(total / (rt60 / (6.0 * np.log(10.0))))
    # directional loudness from a random non-negative-ish order-3 distribution
    # on the 48-point design (sh.py:240-253 formula)
    from .tdesigns import design_for_order
    B = _sh3_np(design_for_order(3).directions)
    D = np.zeros((S, 4, 16, 16))
    for s in range(S):
        for b in range(4):
            avg = rng.normal(scale=0.05, size=16)
            avg[0] = 0.28209479177387814
            g = np.maximum(0.0, B @ avg)
            D[s, b] = (4.0 * np.pi / len(B)) * (B.T * g) @ B
    h_rng = _rng(seed, 1)
    tau = 32.0
    hrtf = (h_rng.standard_normal((16, 2, 256)) * np.exp(-np.arange(256) / tau) / 16.0)
    return dict(dir_direct=d, delay_direct=dist / 343.0 * fs, gain_direct=(1.0 / dist)[:, None] * np.ones((1, 4)),
                predelay=dist / 343.0 * fs + rng.uniform(0.005, 0.02, size=S) * fs,
                fdn_delay=np.round(rng.uniform(0.020, 0.080, size=(S, 16)) * fs).astype(np.int32),
                rt60=rt60, g_reverb=g_reverb, D=D, hrtf=hrtf, hrtf_tau=tau)
