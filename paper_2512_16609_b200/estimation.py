"""Dark channel, atmospheric light, transmission and guided refinement (drop-in for
reference estimation.py:1-172), computed on the GPU (csrc/floatops.cu).

numpy in -> numpy out; CUDA tensors in -> CUDA tensors out.
"""

from __future__ import annotations

from . import floatpath as fp
from .morphology import min_filter
from .validation import check_radius

DEFAULT_PATCH_RADIUS = 7
DEFAULT_TOP_FRACTION = 0.001
DEFAULT_ALPHA = 0.8
DEFAULT_OMEGA = 0.5
DEFAULT_T_MIN = 0.05
DEFAULT_GUIDED_RADIUS = 40
DEFAULT_GUIDED_EPS = 1e-3

# estimation.py:33 — floor applied to airlight components (division safety)
AIRLIGHT_FLOOR = 1e-6


def _out(t, like):
    import torch

    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


def channel_min(image):
    """Per-pixel minimum over the three color channels (estimation.py:35-38)."""
    img = fp.check_float_image(image)
    return _out(fp.channel_min(img), image)


def dark_channel(image, radius=DEFAULT_PATCH_RADIUS):
    """Dark channel: channel minimum eroded over a square patch (estimation.py:41-43)."""
    img = fp.check_float_image(image)
    r = check_radius(radius)
    return _out(fp.min_filter(fp.channel_min(img), r), image)


def estimate_airlight(image, dark, top_fraction=DEFAULT_TOP_FRACTION, alpha=DEFAULT_ALPHA):
    """Atmospheric light from the brightest dark-channel pixels (estimation.py:46-84).

    K = max(1, floor(top_fraction * N)); ties broken by smaller flat index;
    mean RGB (sequential float64 accumulation in selection order) * alpha,
    floored at 1e-6.  Returns a float64 vector of shape (3,).
    """
    img = fp.check_float_image(image)
    d = fp.check_scalar_map(dark, name="dark")
    fp.check_same(img, d, "image", "dark")
    if not 0.0 < top_fraction <= 1.0:
        raise ValueError(f"top_fraction must lie in (0, 1], got {top_fraction}")
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"alpha must lie in (0, 1], got {alpha}")
    return _out(fp.airlight(img, d, top_fraction, alpha), image)


def transmission_from_channel_min(cmin, airlight, omega=DEFAULT_OMEGA, t_min=DEFAULT_T_MIN):
    """t = clip(1 - omega * cmin / max(A), t_min, 1) (estimation.py:87-101)."""
    c = fp.check_scalar_map(cmin, name="cmin")
    a = fp.airlight_tensor(airlight, c.device)
    if not 0.0 < omega <= 1.0:
        raise ValueError(f"omega must lie in (0, 1], got {omega}")
    if not 0.0 < t_min < 1.0:
        raise ValueError(f"t_min must lie in (0, 1), got {t_min}")
    return _out(fp.transmission(c, a, omega, t_min), cmin)


def estimate_transmission(image, airlight, omega=DEFAULT_OMEGA, t_min=DEFAULT_T_MIN):
    """Transmission map for a frame given its atmospheric light (estimation.py:104-107)."""
    img = fp.check_float_image(image)
    a = fp.airlight_tensor(airlight, img.device)
    if not 0.0 < omega <= 1.0:
        raise ValueError(f"omega must lie in (0, 1], got {omega}")
    if not 0.0 < t_min < 1.0:
        raise ValueError(f"t_min must lie in (0, 1), got {t_min}")
    return _out(fp.transmission(fp.channel_min(img), a, omega, t_min), image)


def box_filter(m, radius):
    """Mean over a (2r+1)^2 window, replicate border (estimation.py:110-125).

    Window sums run as sliding sums in runs of 32 outputs (radius-independent
    cost), float64 throughout, divided by k^2 like the reference's SAT.
    """
    t = fp.check_scalar_map(m)
    r = check_radius(radius)
    return _out(fp.box_filter(t, r), m)


def box_filter_naive(m, radius):
    """Per-pixel window mean (reference estimation.py:128-141): an independent device kernel
    (each output sums its own edge-padded window), the reference's correctness check of
    box_filter."""
    t = fp.check_scalar_map(m)
    r = check_radius(radius)
    return _out(fp.box_filter_naive(t, r), m)


def guided_filter(p, guide, radius=DEFAULT_GUIDED_RADIUS, eps=DEFAULT_GUIDED_EPS):
    """Guided filter of map p steered by a grayscale guide, clamped to [0, 1] (estimation.py:144-172)."""
    pt = fp.check_scalar_map(p, name="p")
    gt = fp.check_scalar_map(guide, name="guide")
    fp.check_same(pt, gt, "p", "guide")
    r = check_radius(radius, minimum=1)
    if not eps > 0.0:
        raise ValueError(f"eps must be positive, got {eps}")
    return _out(fp.guided_filter(pt, gt, r, eps), p)


__all__ = [
    "AIRLIGHT_FLOOR",
    "DEFAULT_ALPHA",
    "DEFAULT_GUIDED_EPS",
    "DEFAULT_GUIDED_RADIUS",
    "DEFAULT_OMEGA",
    "DEFAULT_PATCH_RADIUS",
    "DEFAULT_TOP_FRACTION",
    "DEFAULT_T_MIN",
    "box_filter",
    "box_filter_naive",
    "channel_min",
    "dark_channel",
    "estimate_airlight",
    "estimate_transmission",
    "guided_filter",
    "min_filter",
    "transmission_from_channel_min",
]
