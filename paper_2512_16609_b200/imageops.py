"""Pixel format conversion, grayscale and bilinear resizing (drop-in for reference
imageops.py:1-78), computed on the GPU (csrc/floatops.cu)."""

from __future__ import annotations

from . import floatpath as fp
from .validation import check_u8_frame

# Rec.601 luma weights used for the grayscale guide image (imageops.py:15).
GRAY_WEIGHTS = (0.299, 0.587, 0.114)


def _out(t, like):
    import torch

    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


def u8_to_float(frame):
    """uint8 (H, W, 3) -> float64 in [0, 1], true division by 255."""
    import torch

    f = check_u8_frame(frame)
    t = f if isinstance(f, torch.Tensor) else torch.from_numpy(f)
    if not t.is_cuda:
        t = t.to(fp._dev())
    return _out(fp.u8_to_float(t.contiguous()), frame)


def float_to_u8(image):
    """Clamp to [0, 1], *255, +0.5, floor -> uint8 (out-of-range input is legal here)."""
    t = fp.check_float_image(image, clip=True)
    return _out(fp.float_to_u8(t), image)


def to_grayscale(image):
    """Rec.601 luma, clipped to [0, 1]."""
    t = fp.check_float_image(image)
    return _out(fp.to_grayscale(t), image)


def resize_bilinear(image, width, height):
    """Pixel-centre bilinear resize; the identity size returns a copy."""
    t = fp.check_float_image(image)
    width = int(width)
    height = int(height)
    if width < 1 or height < 1:
        raise ValueError(f"target size must be positive, got {width}x{height}")
    return _out(fp.resize_bilinear(t, width, height), image)
