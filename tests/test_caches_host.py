"""Host logic on CPU: the diffuse path (ER) cache with expiry
 and render_early's path prioritization (SPEC.md:400,
437), with the SPEC's own examples."""
import math

import numpy as np

from paper_1803_00430_b200.propagation import CoherenceCaches, PathList
from paper_1803_00430_b200.render import prioritize_paths


def _paths(energies, keys, delays=None):
    n = len(energies)
    E = np.asarray(energies, float).reshape(n, -1)
    return PathList(delays=np.asarray(delays if delays is not None else np.full(n, 0.01)),
                    pressures=np.sqrt(E), directivities=np.tile(np.eye(9)[0], (n, 1)),
                    kinds=["early-reflection"] * n,
                    sources=np.array([k[0] for k in keys], np.int64),
                    orders=np.array([k[1] for k in keys], np.int64),
                    triangles=np.array([[k[2], k[3]] for k in keys], np.int64))


def test_truncation_rule_150_equal_paths():
    """150 equal paths -> exactly 100 rendered, 50 dropped."""
    p = _paths(np.full((150, 4), 1e-6), [(0, 1, i, -1) for i in range(150)])
    kept, dropped = prioritize_paths(p)
    assert len(kept) == 100 and kept.dropped == 50 and len(dropped) == 50
    assert np.array_equal(kept.triangles[:, 0], np.arange(100))        # stable order


def test_threshold_and_sorting():
    inten = np.array([5e-13, 2e-9, 1e-12, 7e-6, 3e-9])
    p = _paths(np.repeat(inten[:, None] / 4, 4, axis=1), [(0, 1, i, -1) for i in range(5)])
    kept, dropped = prioritize_paths(p, max_paths=2)
    assert list(kept.triangles[:, 0]) == [3, 4]                        # loudest first
    assert sorted(dropped.triangles[:, 0]) == [0, 1, 2]                # below threshold or truncated
    kept, _ = prioritize_paths(p, max_paths=10)
    assert 0 not in kept.triangles[:, 0] and 2 in kept.triangles[:, 0]  # 1e-12 is audible


def test_er_cache_smoothing_decay_and_expiry():
    c = CoherenceCaches(tau_er=1.0)
    k1, k2 = (0, 1, 5, -1), (0, 2, 5, 9)
    dt = 1.0
    a = 1.0 - math.exp(-1.0)                                           # SPEC example: dt = tau
    out = c.update_er(_paths([[1.0, 2.0, 3.0, 4.0]], [k1]), dt)        # first sight: taken as is
    assert np.allclose(out.pressures[0] ** 2, [1, 2, 3, 4])
    out = c.update_er(_paths([[2.0, 2.0, 2.0, 2.0], [1.0, 1.0, 1.0, 1.0]], [k1, k2]), dt)
    e1 = out.pressures[[tuple(t) == (5, -1) for t in out.triangles]][0] ** 2
    assert np.allclose(e1, a * 2.0 + (1 - a) * np.array([1, 2, 3, 4]))
    # k1 missing from the next frames: decays, then expires after 2 tau without refresh
    out = c.update_er(_paths([[1.0] * 4], [k2]), dt)
    e1b = out.pressures[[tuple(t) == (5, -1) for t in out.triangles]][0] ** 2
    assert np.allclose(e1b, (1 - a) * e1)
    c.update_er(_paths([[1.0] * 4], [k2]), dt)
    out = c.update_er(_paths([[1.0] * 4], [k2]), dt)
    assert [tuple(t) for t in out.triangles] == [(5, 9)]               # k1 expired
    # a constant path converges to its frame value
    for _ in range(10):
        out = c.update_er(_paths([[1.0] * 4], [k2]), dt)
    assert np.allclose(out.pressures[0] ** 2, 1.0, atol=1e-3)
