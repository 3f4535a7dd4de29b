"""Shared helpers of the GPU parity tests (histogram comparison, ray
selection by a recorded GPU pre-pass, near-tie classification)."""
import numpy as np

HIST_RTOL = 1e-4


def hist_close(Hg, Ho, require_signal=True):
    """1e-4 relative per bin on bins with > 1e-6 of the band's energy
    (BASELINE north_star).  With ``require_signal`` both sides must carry
    energy -- a zero-vs-zero comparison proves nothing."""
    Hg = np.asarray(Hg, np.float64)
    Ho = np.asarray(Ho, np.float64)
    if require_signal:
        assert np.abs(Ho).sum() > 0 and np.abs(Hg).sum() > 0, "vacuous histogram comparison"
    for b in range(Ho.shape[-2]):
        tot = np.abs(Ho[..., b, 0]).sum()
        if tot == 0:
            assert np.abs(Hg[..., b, :]).max() == 0
            continue
        sig = np.abs(Ho[..., b, 0]) > 1e-6 * tot
        for k in range(Ho.shape[-1]):
            a, r = Hg[..., b, k][sig], Ho[..., b, k][sig]
            scale = np.maximum(np.abs(r), np.abs(Ho[..., b, 0][sig]))
            assert np.all(np.abs(a - r) <= HIST_RTOL * scale), (b, k)


def arriving_rays(scene, cfg, sources, keys, listener, n_rays_norm, scan, want, chunk=1 << 16):
    """(source index, global ray indices) pairs whose paths reach the
    listener (recorded GPU pre-pass): chunks of rays of ALL sources are
    traced in one launch each, and the sources with arrivals in a chunk are
    bisected down to single rays with a one-source tracer.  The
    counter-based RNG makes any subset reproducible, so the oracle can trace
    exactly these rays.  Returns {source index: uint32 ray ids}, at most
    ``want`` rays in total."""
    import torch

    from paper_1803_00430_b200 import propagation
    allt = propagation.FrameTracer(scene, len(sources), cfg)
    allt.set_sources(sources, keys)
    one = propagation.FrameTracer(scene, 1, cfg)

    def arrivals_one(a, n):
        one.trace(listener, ray0=a, n_rays=n, total_rays=n_rays_norm)
        torch.cuda.synchronize()
        return int(one.stats[0, 3])

    found = {}
    total = 0
    for a in range(0, scan, chunk):
        n = min(chunk, scan - a)
        allt.trace(listener, ray0=a, n_rays=n, total_rays=n_rays_norm)
        torch.cuda.synchronize()
        per_src = allt.stats[:, 3].cpu().numpy()
        for s in np.nonzero(per_src > 0)[0]:
            one.set_sources(np.asarray(sources)[[s]], [int(keys[s])])
            todo = [(a, n)]
            while todo:
                b, m = todo.pop()
                if m == 1:
                    found.setdefault(int(s), []).append(b)
                    total += 1
                    continue
                h = m // 2
                for c, k in ((b, h), (b + h, m - h)):
                    if arrivals_one(c, k) > 0:
                        todo.append((c, k))
        if total >= want:
            break
    return {s: np.array(sorted(r), np.uint32) for s, r in found.items()}


def mt_uvt(o, d, v0, e1, e2):
    """Moeller-Trumbore (bvh.py:17-27) of one ray and one triangle in numpy
    f64: (t, u, v, det)."""
    p = np.cross(d, e2)
    det = float(e1 @ p)
    if abs(det) <= 1e-14:
        return np.inf, -1.0, -1.0, det
    inv = 1.0 / det
    tv = o - v0
    u = float(tv @ p) * inv
    q = np.cross(tv, e1)
    v = float(q @ d) * inv
    t = float(e2 @ q) * inv
    return t, u, v, det


def edge_margin(o, d, v0, e1, e2):
    t, u, v, _ = mt_uvt(o, d, v0, e1, e2)
    return t, min(u, v, 1.0 - u - v)


def is_documented_near_tie(o, d, tri_a, tri_b, v0, e1, e2, t_limit=None):
    """DESIGN.md 3.2 / SURVEY.md 8(c) exclusions for a ray whose two answers
    (triangle ids, -1 = miss) differ: a hit within 1e-6 (barycentric) of an
    edge on either side, an exact t tie (relative gap < 1e-12), or -- for
    visibility -- a blocker t within 1e-12 of the segment limit."""
    ts = []
    for tri in (tri_a, tri_b):
        if tri < 0:
            continue
        t, m = edge_margin(o, d, v0[tri], e1[tri], e2[tri])
        if abs(m) < 1e-6:
            return True
        ts.append(t)
    if len(ts) == 2 and abs(ts[0] - ts[1]) <= 1e-12 * max(abs(ts[0]), abs(ts[1])):
        return True
    if t_limit is not None and any(abs(t - t_limit) <= 1e-12 * max(abs(t_limit), 1.0) for t in ts):
        return True
    return False
