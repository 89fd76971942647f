"""Scene radiance recovery and post-processing (drop-in for reference recover.py:1-69),
computed on the GPU (csrc/floatops.cu)."""

from __future__ import annotations

from . import floatpath as fp

DEFAULT_GAMMA = 1.2
_MEAN_FLOOR = 1e-6          # recover.py:20
_GAIN_LO, _GAIN_HI = 0.5, 2.0  # recover.py:23-24


def _out(t, like):
    import torch

    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


def recover_radiance(image, airlight, transmission):
    """J = (I - A) / t + A, clamped to [0, 1]; t must be strictly positive."""
    img = fp.check_float_image(image)
    a = fp.airlight_tensor(airlight, img.device)
    t = fp.check_scalar_map(transmission, name="transmission")
    fp.check_same(img, t, "image", "transmission")
    _, lo, _ = fp.stats(t)
    if lo <= 0.0:
        raise ValueError("transmission must be strictly positive everywhere")
    return _out(fp.recover(img, a, t), image)


def gamma_correct(image, gamma=DEFAULT_GAMMA):
    """s -> s**(1/gamma) per sample (a copy when gamma == 1); gamma > 1 brightens."""
    if not gamma > 0.0:
        raise ValueError(f"gamma must be positive, got {gamma}")
    img = fp.check_float_image(image)
    return _out(fp.gamma(img, gamma), image)


def gray_world_balance(image):
    """Scale each channel toward the global mean, gains clipped to [0.5, 2]."""
    img = fp.check_float_image(image)
    return _out(fp.gray_world(img), image)
