"""Real spherical harmonics -- drop-in for echoforge.sh (sh.py).

Basis, ACN ordering and sign convention identical to the reference
(sh.py:1-26): ``eval_sh_batch`` is bit-identical (device kernel with numpy's
expression trees, compiled without FMA contraction).  Batched device
versions: ``eval_sh_batch`` (sh.py:86), ``directional_loudness_matrix`` /
``directional_loudness_batch`` (sh.py:240-253).

``sh_rotation`` builds J(R) by exact quadrature on the 240-point t-design
(degree 21 >= 2*MAX_ORDER) instead of the reference's degree recursion
(sh.py:154-219): J_ij = (4 pi / N) sum_n Y_i(R d_n) Y_j(d_n), which equals the
recursion's matrix to ~1e-14 because both are the unique linear map with
J Y(d) = Y(R d).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .tdesigns import TDesign, design_for_order, tdesign  # noqa: F401

MAX_ORDER = 4

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
         -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
         -0.5900435899266435)
SH_C4 = (2.5033429417967046, -1.7701307697799304, 0.9461746957575601,
         -0.6690465435572892, 0.10578554691520431, -0.6690465435572892,
         0.47308734787878004, -1.7701307697799304, 0.6258357354491761)


def n_coeffs(order: int) -> int:
    return (order + 1) ** 2


def _check_order(order):
    if order < 0 or order > MAX_ORDER:
        raise ValueError(f"order must be in [0, {MAX_ORDER}], got {order}")


class SHVector:
    """Coefficient vector of a real SH expansion (sh.py:33-54)."""

    __slots__ = ("order", "coeffs")

    def __init__(self, order: int, coeffs):
        coeffs = np.asarray(coeffs, dtype=np.float64)
        if coeffs.shape != (n_coeffs(order),):
            raise ValueError(f"order {order} needs {n_coeffs(order)} coefficients, "
                             f"got {coeffs.shape}")
        if not np.all(np.isfinite(coeffs)):
            raise ValueError("non-finite SH coefficients")
        self.order = order
        self.coeffs = coeffs

    @classmethod
    def from_direction(cls, direction, order: int) -> "SHVector":
        return cls(order, eval_sh(direction, order))

    def __repr__(self):
        return f"SHVector(order={self.order}, coeffs={self.coeffs!r})"


class SHRotation:
    """Block-diagonal rotation acting on SH coefficient vectors (sh.py:57-67)."""

    __slots__ = ("order", "matrix")

    def __init__(self, order: int, matrix: np.ndarray):
        self.order = order
        self.matrix = matrix

    def apply(self, coeffs: np.ndarray) -> np.ndarray:
        return self.matrix @ np.asarray(coeffs, dtype=np.float64)


def _check_direction(direction):
    d = np.asarray(direction, dtype=np.float64)
    if d.shape != (3,):
        raise ValueError("direction must be a 3-vector")
    norm = np.linalg.norm(d)
    if abs(norm - 1.0) > 1e-3:
        raise ValueError(f"direction norm {norm:.6g} too far from unit")
    return d / norm


def eval_sh(direction, order: int) -> np.ndarray:
    """SH basis at one unit direction (sh.py:80-83)."""
    return eval_sh_batch(_check_direction(direction)[None, :], order)[0]


def eval_sh_batch(directions, order: int):
    """(N,3) unit directions -> (N,(n+1)^2) on the device (sh.py:86-126).
    numpy in -> numpy out; CUDA tensor in -> CUDA tensor out."""
    _check_order(order)
    t = _lib.torch()
    is_np = not (isinstance(directions, t.Tensor) and directions.is_cuda)
    d = _lib.to_device(directions, t.float64, (-1, 3))
    out = t.empty((d.shape[0], n_coeffs(order)), dtype=t.float64, device=d.device)
    _lib.check(_lib.lib().ef_eval_sh_batch(_lib.ptr(d), d.shape[0], order, _lib.ptr(out),
                                           _lib.stream_handle()))
    return out.cpu().numpy() if is_np else out


def dominant_direction(v) -> np.ndarray | None:
    """normalize(-X_11, -X_1-1, X_10) or None when isotropic (sh.py:129-142)."""
    coeffs = v.coeffs if isinstance(v, SHVector) else np.asarray(v, np.float64)
    if coeffs.shape[0] < 4:
        raise ValueError("dominant_direction needs order >= 1 coefficients")
    vec = np.array([-coeffs[3], -coeffs[1], coeffs[2]])
    norm = np.linalg.norm(vec)
    if norm <= 1e-12 * max(1.0, abs(coeffs[0])):
        return None
    return vec / norm


def _check_rotation(R):
    R = np.asarray(R, dtype=np.float64)
    if R.shape != (3, 3):
        raise ValueError("rotation must be a 3x3 matrix")
    if np.abs(R @ R.T - np.eye(3)).max() > 1e-9 or np.linalg.det(R) < 0:
        raise ValueError("matrix is not a proper rotation")
    return R


def sh_rotation(R, order: int) -> SHRotation:
    """SH-domain rotation J(R) with J(R) Y(d) = Y(R d) (sh.py:154-219)."""
    R = _check_rotation(R)
    _check_order(order)
    design = tdesign(21).directions
    B = eval_sh_batch(design, order)
    BR = eval_sh_batch(design @ R.T, order)
    J = (4.0 * np.pi / len(design)) * (BR.T @ B)
    # exact zeros between degrees
    for l in range(order + 1):
        for l2 in range(order + 1):
            if l != l2:
                J[l * l:(l + 1) ** 2, l2 * l2:(l2 + 1) ** 2] = 0.0
    return SHRotation(order, J)


def sh_transform(directions: np.ndarray, values: np.ndarray, order: int) -> np.ndarray:
    """Least-squares SH fit of sampled sphere values (sh.py:222-237)."""
    dirs = np.asarray(directions, dtype=np.float64)
    vals = np.asarray(values, dtype=np.float64)
    nc = n_coeffs(order)
    if dirs.shape[0] < nc:
        raise ValueError(f"need at least {nc} samples for order {order}, got {dirs.shape[0]}")
    B = eval_sh_batch(dirs, order)
    coeffs, *_ = np.linalg.lstsq(B, vals, rcond=None)
    return coeffs


def directional_loudness_batch(avg, order: int):
    """(n, (order+1)^2) distributions -> (n, nk, nk) loudness matrices on the
    device (batched sh.py:240-253)."""
    _check_order(order)
    t = _lib.torch()
    is_np = not (isinstance(avg, t.Tensor) and avg.is_cuda)
    nk = n_coeffs(order)
    a = _lib.to_device(avg, t.float64, (-1, nk))
    design = _lib.to_device(design_for_order(order).directions, t.float64)
    out = t.empty((a.shape[0], nk, nk), dtype=t.float64, device=a.device)
    _lib.check(_lib.lib().ef_loudness_batch(_lib.ptr(a), a.shape[0], order, _lib.ptr(design),
                                            design.shape[0], _lib.ptr(out), _lib.stream_handle()))
    return out.cpu().numpy() if is_np else out


def directional_loudness_matrix(avg_directivity, order: int) -> np.ndarray:
    """(4 pi/N) B^T diag(max(0, B x)) B on design_for_order(order) (sh.py:240-253)."""
    dist = (avg_directivity.coeffs if isinstance(avg_directivity, SHVector)
            else np.asarray(avg_directivity, dtype=np.float64))
    nc = n_coeffs(order)
    if dist.shape[0] != nc:
        # evaluate the distribution at its own order, re-encode at `order`
        d_order = int(np.sqrt(dist.shape[0])) - 1
        full = np.zeros(max(nc, dist.shape[0]))
        full[:dist.shape[0]] = dist
        if dist.shape[0] > nc:
            design = design_for_order(order).directions
            B = eval_sh_batch(design, order)
            g = np.maximum(0.0, eval_sh_batch(design, d_order) @ dist)
            return (4.0 * np.pi / len(design)) * (B.T * g) @ B
        dist = full[:nc]
    return directional_loudness_batch(dist[None, :], order)[0]


def random_scatter_rotation(rng: np.random.Generator) -> np.ndarray:
    """Rz Ry Rx with per-axis angles uniform in [90, 270] deg (sh.py:256-265)."""
    ax, ay, az = rng.uniform(np.pi / 2, 3 * np.pi / 2, size=3)

    def rot(axis, a):
        c, s = np.cos(a), np.sin(a)
        m = np.eye(3)
        i, j = [(1, 2), (0, 2), (0, 1)][axis]
        m[i, i], m[j, j] = c, c
        m[i, j], m[j, i] = -s, s
        if axis == 1:
            m[i, j], m[j, i] = s, -s
        return m

    return rot(2, az) @ rot(1, ay) @ rot(0, ax)
