"""Grayscale erosion over a square window (drop-in for reference morphology.py:63-92).

The reference uses van Herk/Gil-Werman running minima; min only selects, so any
evaluation order is bit-identical.  The device kernels (csrc/floatops.cu) take
the clamped-window minimum, rows then columns.
"""

from __future__ import annotations

from . import floatpath as fp
from .validation import check_radius


def _out(t, like):
    import torch

    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


def min_filter(m, radius):
    """Erode a 2-D map with a (2*radius+1) square window, replicate border."""
    t = fp.check_scalar_map(m)
    r = check_radius(radius)
    return _out(fp.min_filter(t, r), m)


def min_filter_naive(m, radius):
    """Per-pixel window scan (reference morphology.py:76-92): an independent device kernel
    (every output scans its own clamped window), the reference's correctness check of
    min_filter."""
    t = fp.check_scalar_map(m)
    r = check_radius(radius)
    return _out(fp.min_filter_naive(t, r), m)
