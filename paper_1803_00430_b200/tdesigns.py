"""Embedded spherical t-designs -- drop-in for echoforge.tdesigns.

The point tables (degrees 3/5/9/21 -> 6/12/48/240 directions) are data
exported from the reference by oracle/gen_golden.py into data/tdesigns.npz
(tdesigns.py:14-330); the selection rules follow tdesigns.py:351-362.
"""
from __future__ import annotations

import os

import numpy as np

__all__ = ["TDesign", "tdesign", "design_for_order", "AVAILABLE_DEGREES"]

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "tdesigns.npz")
with np.load(_DATA) as _z:
    _TABLES = {int(k[1:]): np.array(_z[k]) for k in _z.files}
AVAILABLE_DEGREES = tuple(sorted(_TABLES))


class TDesign:
    """Unit directions with equal quadrature weight, exact to degree t."""

    def __init__(self, degree: int, directions: np.ndarray):
        directions = np.asarray(directions, dtype=np.float64)
        if np.abs(np.linalg.norm(directions, axis=1) - 1.0).max() > 1e-12:
            raise ValueError("t-design directions must be unit vectors")
        self.degree = degree
        self.directions = directions

    def __len__(self) -> int:
        return len(self.directions)


def tdesign(degree: int) -> TDesign:
    """Smallest embedded design whose degree is >= the requested degree."""
    for t in AVAILABLE_DEGREES:
        if t >= degree:
            return TDesign(t, _TABLES[t])
    raise ValueError(f"no embedded t-design of degree >= {degree} (available: {AVAILABLE_DEGREES})")


def design_for_order(order: int) -> TDesign:
    """Design exact for products of two order-n functions (degree 2n+1)."""
    return tdesign(2 * order + 1)
