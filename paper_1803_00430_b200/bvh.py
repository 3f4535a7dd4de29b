"""Ray-triangle queries -- drop-in for echoforge.bvh (bvh.py).

``ray_triangles`` / ``ray_triangles_batch`` run the reference's
Moeller-Trumbore arithmetic (bvh.py:11-45) on the GPU with numpy's exact
evaluation order, returning the same (t, valid) arrays.  ``BVH`` keeps the
reference constructor and ``intersect(origin, direction, t_min, t_max)``
(bvh.py:51, 130) but the tree lives on the device (csrc/bvh_build.cpp) and the
query is a device kernel.

One documented difference: the reference computes ``v`` on its per-ray path
with OpenBLAS (``qvec @ direction``, bvh.py:24), whose FMA order depends on
the host CPU; the device uses numpy-einsum order everywhere.  Only hits within
~1 ulp of a triangle edge can differ (near-ties).
"""
from __future__ import annotations

import numpy as np

from . import _lib

_LEAF_SIZE = 4          # bvh.py:6 (reference builder; the device builder uses <= 4 too)
_N_BINS = 16            # bvh.py:7 (reference; the device builder bins 32 per axis)
_BARY_EPS = 1e-10       # bvh.py:8


def _as_rays(a, b):
    """Two (n,3) f64 inputs -> device tensors; remembers whether to return numpy."""
    t = _lib.torch()
    is_np = not (isinstance(a, t.Tensor) and a.is_cuda)
    return _lib.to_device(a, t.float64, (-1, 3)), _lib.to_device(b, t.float64, (-1, 3)), is_np


def _out(tensors, is_np):
    if not is_np:
        return tensors
    return tuple(x.cpu().numpy() for x in tensors)


def _ray_triangles_dev(origins, directions, v0, e1, e2, t_min, t_max):
    t = _lib.torch()
    o, d, is_np = _as_rays(origins, directions)
    V0, E1, _ = _as_rays(v0, e1)
    E2 = _lib.to_device(e2, t.float64, (-1, 3))
    nr, nt = o.shape[0], V0.shape[0]
    tt = t.empty((nr, nt), dtype=t.float64, device=o.device)
    valid = t.empty((nr, nt), dtype=t.uint8, device=o.device)
    tm = None
    if t_max is not None:
        tm = _lib.to_device(np.broadcast_to(np.asarray(t_max, np.float64), (nr,)), t.float64)
    _lib.check(_lib.lib().ef_ray_triangles(_lib.ptr(o), _lib.ptr(d), nr, _lib.ptr(V0),
                                           _lib.ptr(E1), _lib.ptr(E2), nt, float(t_min),
                                           _lib.ptr(tm), _lib.ptr(tt), _lib.ptr(valid),
                                           _lib.stream_handle()))
    return _out((tt, valid.bool()), is_np)


def ray_triangles(origin, direction, v0, e1, e2, t_min, t_max):
    """One ray against a triangle array: (t, valid) of shape (K,) (bvh.py:11-28)."""
    t, valid = _ray_triangles_dev(np.asarray(origin, np.float64).reshape(1, 3),
                                  np.asarray(direction, np.float64).reshape(1, 3),
                                  v0, e1, e2, t_min, t_max)
    return t[0], valid[0]


def ray_triangles_batch(origins, directions, v0, e1, e2, t_min):
    """All rays against all triangles: (t, valid) of shape (R, T) (bvh.py:31-45)."""
    return _ray_triangles_dev(origins, directions, v0, e1, e2, t_min, None)


class BVH:
    """Device BVH over a triangle soup (bvh.py:48-160).

    ``BVH(v0, e1, e2)`` builds on first use; ``intersect`` returns
    ``(t, triangle_id)`` or ``(inf, -1)``.  Constructing it from a SceneModel
    shares that scene's device handle.
    """

    def __init__(self, v0: np.ndarray, e1: np.ndarray, e2: np.ndarray, _scene=None):
        self.v0, self.e1, self.e2 = v0, e1, e2
        self.n_triangles = len(v0)
        self._scene = _scene

    def _model(self):
        if self._scene is None:
            from .scene import Listener, Material, SceneModel, Source
            self._scene = SceneModel(self.v0, self.e1, self.e2, np.zeros(self.n_triangles, np.int64),
                                     [Material("bvh", [0.0], [0.0])],
                                     [Source(id="bvh", position=np.zeros(3))],
                                     Listener(position=np.zeros(3)))
        return self._scene

    def intersect(self, origin, direction, t_min, t_max):
        """Nearest hit in (t_min, t_max]: (t, triangle_id) or (inf, -1)."""
        if self.n_triangles == 0:
            return np.inf, -1
        t, tri, hit = self._model()._query(np.asarray(origin, np.float64).reshape(1, 3),
                                           np.asarray(direction, np.float64).reshape(1, 3),
                                           t_min, t_max, 2)
        if not hit[0]:
            return np.inf, -1
        return float(t[0]), int(tri[0])

    def intersect_batch(self, origins, directions, t_min, t_max=None):
        """Batched ``intersect`` (one kernel launch for all rays)."""
        return self._model()._query(origins, directions, t_min, t_max, 2)
