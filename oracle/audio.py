"""CPU oracle of the SH-domain auralization (config C4) -- TEST
INFRASTRUCTURE ONLY (tests/ and bench.py's CPU leg).

The reference ships no renderer code; this restates, in float64 numpy/scipy,
the pinned block semantics of DESIGN.md section 3.7 (SPEC.md:361-450 reverb
renderer with BASELINE C4's 16-line FDN per band; SPEC.md:452-517 binaural
decode), "parity unpinned" beyond the SPEC's own examples:

  crossover     LR4 tree at 176 / 775 / 3408 Hz with allpass compensation
                (SPEC.md:366-369, 388-396), RBJ biquads, state carried over
  delay taps    per-band circular history, linear fractional interpolation
                
  direct path   tap at the direct delay, gain a_b, SH encode Y(dir) order 3
  reverb send   tap at the predelay into a 16-line FDN per band, Householder
                feedback, per-line gains 10^(-3 m_i / (fs RT60_b)) (Eq. 7,
                SPEC.md:412), lines -> SH via g_reverb,b * D_b * E
  binaural      q_ear = sum_k bus_k (*) h_k,ear, here as a full direct
                convolution; the device uses overlap-save
"""
from __future__ import annotations

import numpy as np
from scipy import signal

FS = 48000.0
BLOCK = 512
N_LINES = 16
EDGES = (176.0, 775.0, 3408.0)


def rbj(kind: str, f0: float, fs: float = FS, q: float = 1.0 / np.sqrt(2.0)) -> np.ndarray:
    """One RBJ-cookbook biquad as an SOS row [b0 b1 b2 1 a1 a2] (a0-normalised)."""
    w0 = 2.0 * np.pi * f0 / fs
    c, s = np.cos(w0), np.sin(w0)
    alpha = s / (2.0 * q)
    if kind == "lp":
        b = [(1 - c) / 2, 1 - c, (1 - c) / 2]
    elif kind == "hp":
        b = [(1 + c) / 2, -(1 + c), (1 + c) / 2]
    elif kind == "ap":
        b = [1 - alpha, -2 * c, 1 + alpha]
    else:
        raise ValueError(kind)
    a = [1 + alpha, -2 * c, 1 - alpha]
    return np.array([b[0] / a[0], b[1] / a[0], b[2] / a[0], 1.0, a[1] / a[0], a[2] / a[0]])


def band_sos() -> list[np.ndarray]:
    """Per band the cascade: LR4 (two identical Butterworth biquads) at the
    middle split, LR4 at the outer split, allpass at the other outer split."""
    f1, f2, f3 = EDGES
    lp = lambda f: [rbj("lp", f), rbj("lp", f)]  # noqa: E731
    hp = lambda f: [rbj("hp", f), rbj("hp", f)]  # noqa: E731
    return [np.array(lp(f2) + lp(f1) + [rbj("ap", f3)]),
            np.array(lp(f2) + hp(f1) + [rbj("ap", f3)]),
            np.array(hp(f2) + lp(f3) + [rbj("ap", f1)]),
            np.array(hp(f2) + hp(f3) + [rbj("ap", f1)])]


def line_directions() -> np.ndarray:
    """16-point spherical Fibonacci set (directions of the FDN lines)."""
    i = np.arange(N_LINES)
    z = 1.0 - (2.0 * i + 1.0) / N_LINES
    r = np.sqrt(1.0 - z * z)
    phi = i * np.pi * (3.0 - np.sqrt(5.0))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def eval_sh3(d):
    """Order-3 real SH (sh.py:86-126 formulas), f64."""
    from oracle.oracle import eval_sh_batch
    return eval_sh_batch(np.asarray(d, np.float64).reshape(-1, 3), 3)


class AudioOracle:
    """Float64 block renderer for S sources (state carried across blocks)."""

    def __init__(self, p: dict, hrtf: np.ndarray):
        self.p = p
        S = p["dir_direct"].shape[0]
        self.S = S
        self.nb = 4
        self.sos = band_sos()
        self.zi = np.zeros((S, self.nb, 5, 2))
        self.hist = np.zeros((S, self.nb, 0))           # band histories (all samples)
        self.lines = np.zeros((S, self.nb, N_LINES, 0))  # FDN line inputs s_i[n]
        self.Y = eval_sh3(p["dir_direct"])              # (S, 16)
        E = eval_sh3(line_directions()).T * np.sqrt(4.0 * np.pi / N_LINES)   # (16 sh, 16 lines)
        m = p["fdn_delay"].astype(np.float64)           # (S, 16) samples
        self.g_line = 10.0 ** (-3.0 * m[:, None, :] / (FS * p["rt60"][:, :, None]))  # (S,nb,16)
        # per band: SH out = g_reverb,b * D_b @ E  (S, nb, 16 sh, 16 lines)
        self.M = p["g_reverb"][:, :, None, None] * np.einsum("sbkj,ji->sbki", p["D"], E)
        self.hrtf = hrtf                                # (16, 2, taps)
        self.bus_hist = np.zeros((16, 0))

    def update(self, p: dict):
        """update_params at a block boundary: new direct / reverb parameters
        (line delays and HRTF unchanged), state carried over."""
        q = dict(self.p)
        for k in ("dir_direct", "delay_direct", "gain_direct", "predelay", "rt60", "g_reverb", "D"):
            q[k] = p[k]
        self.p = q
        self.Y = eval_sh3(q["dir_direct"])
        E = eval_sh3(line_directions()).T * np.sqrt(4.0 * np.pi / N_LINES)
        m = q["fdn_delay"].astype(np.float64)
        self.g_line = 10.0 ** (-3.0 * m[:, None, :] / (FS * q["rt60"][:, :, None]))
        self.M = q["g_reverb"][:, :, None, None] * np.einsum("sbkj,ji->sbki", q["D"], E)

    @staticmethod
    def tap(hist, start, delay):
        """Linear fractional read of samples [start, start+BLOCK) delayed by
        `delay` (>= 1) from a history array (zeros before time 0)."""
        n = start + np.arange(BLOCK) - delay
        i0 = np.floor(n).astype(np.int64)
        f = n - i0
        def get(i):
            ok = (i >= 0) & (i < hist.shape[-1])
            return np.where(ok, hist[..., np.clip(i, 0, max(hist.shape[-1] - 1, 0))], 0.0)
        return (1.0 - f) * get(i0) + f * get(i0 + 1)

    def process(self, x: np.ndarray):
        """x: (S, BLOCK) float32 input block -> (bus (16, BLOCK), out (2, BLOCK))."""
        S, nb, p = self.S, self.nb, self.p
        start = self.hist.shape[-1]
        bands = np.zeros((S, nb, BLOCK))
        for s in range(S):
            for b in range(nb):
                y, self.zi[s, b] = signal.sosfilt(self.sos[b], x[s].astype(np.float64),
                                                  zi=self.zi[s, b])
                bands[s, b] = y
        self.hist = np.concatenate([self.hist, bands], axis=-1)
        bus = np.zeros((16, BLOCK))
        # direct path
        for s in range(S):
            d = self.tap(self.hist[s], start, p["delay_direct"][s])            # (nb, BLOCK)
            mono = (p["gain_direct"][s][:, None] * d).sum(axis=0)
            bus += self.Y[s][:, None] * mono[None, :]
        # reverb: FDN per band, outputs only depend on previous blocks (m_i > BLOCK)
        new_lines = np.zeros((S, nb, N_LINES, BLOCK))
        for s in range(S):
            send = self.tap(self.hist[s], start, p["predelay"][s])              # (nb, BLOCK)
            m = p["fdn_delay"][s]
            for b in range(nb):
                y = np.zeros((N_LINES, BLOCK))
                for i in range(N_LINES):
                    idx = start + np.arange(BLOCK) - m[i]
                    ok = idx >= 0
                    y[i, ok] = self.lines[s, b, i, idx[ok]]
                gy = self.g_line[s, b][:, None] * y
                fb = gy - (2.0 / N_LINES) * gy.sum(axis=0, keepdims=True)     # Householder
                new_lines[s, b] = 0.25 * send[b][None, :] + fb
                bus += self.M[s, b] @ y
        self.lines = np.concatenate([self.lines, new_lines], axis=-1)
        # binaural: full direct convolution of the bus history
        self.bus_hist = np.concatenate([self.bus_hist, bus], axis=1)
        taps = self.hrtf.shape[-1]
        out = np.zeros((2, BLOCK))
        seg = self.bus_hist[:, max(0, start - taps + 1):]
        off = start - max(0, start - taps + 1)
        for e in range(2):
            acc = np.zeros(seg.shape[1] + taps - 1)
            for k in range(16):
                acc += np.convolve(seg[k], self.hrtf[k, e])
            out[e] = acc[off:off + BLOCK]
        return bus, out
