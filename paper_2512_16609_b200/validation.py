"""Host-side argument contracts (mirror of reference validation.py:17-107).

The drop-in keeps the reference's ValueError texts (its tests match them by
regex: "uint8", "H, W, 3", "finite", "outside", "2-D", "disagree", ...).
Arrays that are already CUDA tensors are checked on the device with a single
fused reduction instead of host scans.
"""

from __future__ import annotations

import numpy as np

RANGE_SLACK = 1e-9  # validation.py:11


def _is_tensor(x):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def check_u8_frame(frame, name="frame"):
    """validation.py:17-29 — (H, W, 3) uint8; returns a C-contiguous array/tensor."""
    if _is_tensor(frame):
        import torch

        if frame.dtype != torch.uint8:
            raise ValueError(f"{name}: expected dtype uint8, got {frame.dtype}")
        shape = tuple(frame.shape)
        if frame.dim() != 3 or shape[2] != 3:
            raise ValueError(f"{name}: expected shape (H, W, 3), got {shape}")
        if shape[0] < 1 or shape[1] < 1:
            raise ValueError(f"{name}: empty image {shape[0]}x{shape[1]}")
        return frame.contiguous()
    arr = np.asarray(frame)
    if arr.dtype != np.uint8:
        raise ValueError(f"{name}: expected dtype uint8, got {arr.dtype}")
    if arr.ndim != 3 or arr.shape[2] != 3:
        raise ValueError(f"{name}: expected shape (H, W, 3), got {arr.shape}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"{name}: empty image {arr.shape[0]}x{arr.shape[1]}")
    return np.ascontiguousarray(arr)


def _range_error(name, lo, hi):
    return ValueError(f"{name}: samples outside [0, 1] (min {lo:.6g}, max {hi:.6g})")


def check_float_image_shape(shape, name="image"):
    if len(shape) != 3 or shape[2] != 3:
        raise ValueError(f"{name}: expected shape (H, W, 3), got {tuple(shape)}")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"{name}: empty image {shape[0]}x{shape[1]}")


def check_scalar_map_shape(shape, name="map"):
    if len(shape) != 2:
        raise ValueError(f"{name}: expected a 2-D map, got shape {tuple(shape)}")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"{name}: empty map {shape[0]}x{shape[1]}")


def check_stats(name, finite, lo, hi, clip, kind="samples"):
    """Shared tail of check_float_image / check_scalar_map given (all-finite, min, max)."""
    if not finite:
        raise ValueError(f"{name}: contains non-finite {kind}")
    if not clip and (lo < -RANGE_SLACK or hi > 1.0 + RANGE_SLACK):
        raise _range_error(name, lo, hi)


def check_airlight(airlight, name="airlight"):
    """validation.py:75-88 — shape (3,), finite, every component in (0, 1]."""
    if _is_tensor(airlight):
        airlight = airlight.detach().cpu().numpy()
    arr = np.asarray(airlight, dtype=np.float64)
    if arr.shape != (3,):
        raise ValueError(f"{name}: expected shape (3,), got {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValueError(f"{name}: contains non-finite components")
    if arr.min() <= 0.0 or arr.max() > 1.0:
        raise ValueError(f"{name}: components must lie in (0, 1], got {arr.tolist()}")
    return arr


def check_radius(radius, name="radius", minimum=0):
    """validation.py:91-98."""
    r = int(radius)
    if r != radius:
        raise ValueError(f"{name}: expected an integer, got {radius!r}")
    if r < minimum:
        raise ValueError(f"{name}: must be >= {minimum}, got {r}")
    return r


def check_same_shape(shape_a, shape_b, name_a, name_b):
    """validation.py:101-107 (on shapes)."""
    if tuple(shape_a[:2]) != tuple(shape_b[:2]):
        raise ValueError(
            f"{name_a} and {name_b} disagree on size: {tuple(shape_a[:2])} vs {tuple(shape_b[:2])}"
        )
