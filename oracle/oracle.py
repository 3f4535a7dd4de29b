"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's
``cpu_baseline`` / ``--impl reference`` legs, as the checker or the CPU
baseline.  The product package ``paper_1803_00430_b200`` never imports it.

Two halves:
  * ``libefo.so`` (oracle/efo.c): the reference's intersection + BVH
    (bvh.py:11-160, scene.py:208-230) restated bit-for-bit, plus the pinned
    bounce loop / listener receiver / SH histogram.
  * numpy restatements of the SPEC-only estimators and of
    the reference's SH helpers (sh.py:86-126, 240-253).

The intersection/BVH/SH parts are pinned against golden vectors produced by
the reference itself (tests/golden, oracle/gen_golden.py).  The bounce loop,
histogram and estimators have no reference code: "parity unpinned" beyond
this restatement and its known-answer tests (SPEC.md examples).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libefo.so")
_lib = None

ST_NAMES = ("paths", "segments", "reflections", "arrivals", "direct", "dropped",
            "escaped", "nodes", "tris", "neartie_paths")

_c_double_p = ctypes.POINTER(ctypes.c_double)


def build():
    """Compile oracle/efo.c (gcc) into oracle/_build/libefo.so."""
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp = ctypes.c_void_p
        L.efo_scene_create.restype = vp
        L.efo_scene_create.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int64, vp, vp,
                                       ctypes.c_int, ctypes.c_int]
        L.efo_scene_destroy.argtypes = [vp]
        L.efo_scene_n_nodes.restype = ctypes.c_int64
        L.efo_scene_n_nodes.argtypes = [vp]
        L.efo_scene_bvh.argtypes = [vp] * 7
        L.efo_material_tables.argtypes = [vp] * 4
        L.efo_intersect_batch.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_double, vp,
                                          ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp]
        L.efo_eval_sh_batch.argtypes = [vp, ctypes.c_int64, ctypes.c_int, vp]
        L.efo_philox.argtypes = [vp, vp, vp]
        L.efo_sample_sphere.argtypes = [ctypes.c_uint32] * 4 + [vp]
        L.efo_trace.argtypes = [vp, vp, ctypes.c_uint32, vp, vp, ctypes.c_uint32,
                                ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int64, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class _TraceCfg(ctypes.Structure):
    _fields_ = [("n_bands", ctypes.c_int32), ("order", ctypes.c_int32),
                ("n_bins", ctypes.c_int32), ("max_bounces", ctypes.c_int32),
                ("bin_len", ctypes.c_double), ("listener", ctypes.c_double * 3),
                ("radius", ctypes.c_double), ("seed", ctypes.c_uint32),
                ("frame", ctypes.c_uint32), ("vmode", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("e0", ctypes.c_float),
                ("rain", ctypes.c_int32), ("er_max_order", ctypes.c_int32)]


class ErEntry(ctypes.Structure):
    _fields_ = [("src", ctypes.c_int32), ("order", ctypes.c_int32), ("tri0", ctypes.c_int32),
                ("tri1", ctypes.c_int32), ("dist", ctypes.c_double), ("dir", ctypes.c_float * 3),
                ("pad", ctypes.c_float), ("energy", ctypes.c_float * 8)]


ER_DTYPE = np.dtype([("src", "<i4"), ("order", "<i4"), ("tri0", "<i4"), ("tri1", "<i4"),
                     ("dist", "<f8"), ("dir", "<f4", 3), ("pad", "<f4"), ("energy", "<f4", 8)])


def philox(ctr, key):
    """Philox4x32-10 of one 128-bit counter under a 64-bit key."""
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().efo_philox(_p(c), _p(k), _p(out))
    return out


def sample_sphere(seed, src, ray, frame=0):
    d = np.zeros(3)
    lib().efo_sample_sphere(seed, src, ray, frame, _p(d))
    return d


def eval_sh_batch(dirs, order):
    """sh.py:86-126 restated in C (same expression trees)."""
    d = _c(dirs, np.float64).reshape(-1, 3)
    out = np.zeros((len(d), (order + 1) ** 2))
    lib().efo_eval_sh_batch(_p(d), len(d), order, _p(out))
    return out


class OracleScene:
    """Triangle soup + the reference's binned-SAH BVH (bvh.py:51-128)."""

    def __init__(self, v0, e1, e2, normals, material_index, absorption, scattering):
        self.v0 = _c(v0, np.float64).reshape(-1, 3)
        self.e1 = _c(e1, np.float64).reshape(-1, 3)
        self.e2 = _c(e2, np.float64).reshape(-1, 3)
        self.normals = _c(normals, np.float64).reshape(-1, 3)
        self.mat = _c(material_index, np.int64)
        self.absorption = _c(absorption, np.float64)
        self.scattering = _c(scattering, np.float64)
        self.n_bands = self.absorption.shape[1]
        self.n_tri = len(self.v0)
        self._h = lib().efo_scene_create(
            _p(self.v0), _p(self.e1), _p(self.e2), _p(self.normals), _p(self.mat),
            self.n_tri, _p(self.absorption), _p(self.scattering),
            self.absorption.shape[0], self.n_bands)

    @classmethod
    def from_arrays(cls, arrays: dict):
        return cls(arrays["v0"], arrays["e1"], arrays["e2"], arrays["normals"],
                   arrays["material_index"], arrays["absorption"], arrays["scattering"])

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.efo_scene_destroy(self._h)
            self._h = None

    def bvh_arrays(self):
        n = lib().efo_scene_n_nodes(self._h)
        nmin = np.zeros((n, 3)); nmax = np.zeros((n, 3))
        left = np.zeros(n, np.int64); start = np.zeros(n, np.int64); count = np.zeros(n, np.int64)
        order = np.zeros(self.n_tri, np.int64)
        lib().efo_scene_bvh(self._h, _p(nmin), _p(nmax), _p(left), _p(start), _p(count), _p(order))
        return dict(node_min=nmin, node_max=nmax, node_left=left, node_start=start,
                    node_count=count, tri_order=order)

    def material_tables(self):
        m, nb = self.absorption.shape
        fd = np.zeros((m, nb), np.float32); fs = np.zeros((m, nb), np.float32)
        pd = np.zeros(m)
        lib().efo_material_tables(self._h, _p(fd), _p(fs), _p(pd))
        return fd, fs, pd

    def intersect_batch(self, origins, directions, t_min=1e-4, t_max=None, mode=0,
                        blas_v=False, counters=False):
        """scene.py:208-230.  mode 0: reference dispatch (brute <= 512 tris
        else BVH), 1: brute, 2: BVH.  Returns (t, tri, hit[, nodes, tris])."""
        o = _c(origins, np.float64).reshape(-1, 3)
        d = _c(directions, np.float64).reshape(-1, 3)
        n = len(o)
        tm = None if t_max is None else _c(np.broadcast_to(t_max, (n,)), np.float64)
        t = np.zeros(n); tri = np.zeros(n, np.int64); hit = np.zeros(n, np.uint8)
        nn = np.zeros(n, np.int64); nt = np.zeros(n, np.int64)
        lib().efo_intersect_batch(self._h, _p(o), _p(d), n, t_min, _p(tm), mode, int(blas_v),
                                  _p(t), _p(tri), _p(hit), _p(nn), _p(nt))
        if counters:
            return t, tri, hit.astype(bool), nn, nt
        return t, tri, hit.astype(bool)


@dataclass
class OracleTrace:
    H: np.ndarray          # (n_bins, n_bands, nk) float64 sums of f32 splats
    Dir: np.ndarray        # (n_bands, nk)
    stats: dict
    sum_t: float
    nseg: np.ndarray | None
    ids: np.ndarray | None
    first_tie: np.ndarray | None
    er: np.ndarray | None = None


def trace(scene: OracleScene, *, src_key, src_pos, listener, radius, seed, frame=0,
          order, n_bins, bin_len, max_bounces, e0, rays=None, ray0=0, n_rays=None,
          record=False, mode=0, blas_v=False, rain=False, er_max_order=0, er_capacity=0):
    """Pinned bounce loop for one source."""
    cfg = _TraceCfg()
    cfg.n_bands = scene.n_bands
    cfg.order = order
    cfg.n_bins = n_bins
    cfg.max_bounces = max_bounces
    cfg.bin_len = bin_len
    cfg.listener[:] = [float(x) for x in listener]
    cfg.radius = radius
    cfg.seed = seed
    cfg.frame = frame
    cfg.vmode = int(blas_v)
    cfg.mode = mode
    cfg.e0 = float(np.float32(e0))
    cfg.rain = int(rain)
    cfg.er_max_order = int(er_max_order)
    if rays is not None:
        rays = _c(rays, np.uint32)
        n = len(rays)
    else:
        n = int(n_rays)
    nk = (order + 1) ** 2
    H = np.zeros((n_bins, scene.n_bands, nk))
    Dir = np.zeros((scene.n_bands, nk))
    st = np.zeros(len(ST_NAMES), np.uint64)
    sum_t = np.zeros(1)
    nseg = np.zeros(n, np.int32) if record else None
    ids = np.full((n, max_bounces), -2, np.int32) if record else None
    ftie = np.zeros(n, np.int32) if record else None
    pos = _c(src_pos, np.float64)
    er = np.zeros(max(er_capacity, 1), ER_DTYPE)
    er_n = np.zeros(1, np.int64)
    lib().efo_trace(scene._h, ctypes.byref(cfg), src_key, _p(pos), _p(rays), ray0, n,
                    _p(H), _p(Dir), _p(st), _p(sum_t), _p(nseg), _p(ids), _p(ftie),
                    _p(er), er_capacity, _p(er_n))
    return OracleTrace(H, Dir, dict(zip(ST_NAMES, (int(x) for x in st))), float(sum_t[0]),
                       nseg, ids, ftie, er[:min(int(er_n[0]), er_capacity)])
