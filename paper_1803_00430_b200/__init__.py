"""paper_1803_00430_b200 -- B200-native hot path of the echoforge reference
(arXiv 1803.00430): seeded ray generation, BVH traversal with the reference's
exact f64 intersection, the bounce loop into SH energy IR histograms, per-band
decay fits and SH loudness -- behind the reference's Python signatures and a
C ABI (include/echoforge_b200.h).  See DESIGN.md."""

__version__ = "0.1.0"

from . import _lib  # noqa: F401
