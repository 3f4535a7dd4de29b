"""CPU oracle of the ir-analysis module -- TEST INFRASTRUCTURE ONLY.

Restates, in plain numpy/f64, the estimator choices pinned in DESIGN.md 3.6
for the SPEC-only operations (no reference code exists; "parity unpinned"
beyond this restatement and the SPEC's own known-answer examples):

  estimate_rt60          SPEC.md:272-280, decisions 344-346
  reverb_gain
  estimate_predelay      SPEC.md:299-307, decision 347
  average_directivity
  directional_loudness   the reference's sh.py:240-253 formula (pinned
                         against the reference itself in tests/golden/sh.npz)
"""
from __future__ import annotations

import math

import numpy as np

Y00 = 0.28209479177387814


def rt60_fit(I, bin_s, max_rt):
    """Returns (rt60, silent, n_fit, slope) for one intensity series."""
    I = np.asarray(I, dtype=np.float64)
    nz = np.nonzero(I > 0.0)[0]
    if len(nz) < 3:
        return 1.0, True, 0, 0.0
    last = nz[-1]
    edc = np.cumsum(I[:last + 1][::-1])[::-1]
    db = 10.0 * np.log10(edc / edc[0])
    x = np.arange(last + 1, dtype=np.float64) * bin_s
    if db[last] <= -35.0:
        lim = -35.0
    elif db[last] <= -25.0:
        lim = -25.0
    else:
        return 1.0, True, 0, 0.0
    sel = (db <= -5.0) & (db >= lim)
    n = int(sel.sum())
    if n < 2:
        return 1.0, True, 0, 0.0
    xs, ys = x[sel], db[sel]
    den = n * np.sum(xs * xs) - np.sum(xs) ** 2
    if not den > 0:
        return 1.0, True, 0, 0.0
    slope = (n * np.sum(xs * ys) - np.sum(xs) * np.sum(ys)) / den
    if not slope < 0:
        return 1.0, True, 0, 0.0
    return float(min(max(-60.0 / slope, 0.05), max_rt)), False, n, float(slope)


def reverb_gain(total, rt60):
    return math.sqrt(total / (rt60 / (6.0 * math.log(10.0)))) if total > 0 else 0.0


def loudness(avg, B):
    g = np.maximum(0.0, B @ avg)
    return (4.0 * np.pi / len(B)) * (B.T * g) @ B


def analyze(H, Dir, sum_t, n_reflections, bin_s, max_rt, B=None):
    """H: (n_bins, n_bands, nk) energy histogram of ONE source (f32 or f64);
    Dir: (n_bands, nk).  Returns a dict of per-band arrays and scalars."""
    H = np.asarray(H, dtype=np.float64)
    Dir = np.asarray(Dir, dtype=np.float64)
    nb = H.shape[1]
    out = {k: np.zeros(nb) for k in ("rt60", "gain", "drr_db", "total", "direct", "silent",
                                     "fit_n", "slope")}
    out["avg"] = np.zeros((nb, H.shape[2]))
    out["loudness"] = None if B is None else np.zeros((nb, H.shape[2], H.shape[2]))
    first = None
    for b in range(nb):
        I = H[:, b, 0] / Y00
        rt, silent, n, slope = rt60_fit(I, bin_s, max_rt)
        total = float(H[:, b, 0].sum() / Y00)
        edir = float(Dir[b, 0] / Y00)
        if not edir > 0:
            drr = -99.0
        elif not total > 0:
            drr = 99.0
        else:
            drr = float(np.clip(10.0 * np.log10(edir / total), -99.0, 99.0))
        out["rt60"][b] = rt
        out["gain"][b] = reverb_gain(total, rt) if not silent else 0.0
        out["drr_db"][b] = drr
        out["total"][b] = total
        out["direct"][b] = edir
        out["silent"][b] = float(silent)
        out["fit_n"][b] = n
        out["slope"][b] = slope
        avg = H[:, b, :].sum(axis=0) / total if total > 0 else np.zeros(H.shape[2])
        out["avg"][b] = avg
        if B is not None:
            out["loudness"][b] = loudness(avg, B)
        nzb = np.nonzero(I > 0.0)[0]
        if len(nzb):
            first = nzb[0] if first is None else min(first, nzb[0])
    out["predelay"] = -1.0 if first is None else first * bin_s
    out["mfp"] = sum_t / n_reflections if n_reflections else 0.0
    return out
