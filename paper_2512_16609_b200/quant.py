"""Exact output-byte thresholds for the recover -> gamma -> quantise chain.

The reference maps a recovered sample ``x`` in [0, 1] to its output byte with

    y = clip(power(x, 1/gamma), 0, 1)        (recover.py:51-54; a copy when gamma == 1)
    q = floor(clip(y, 0, 1) * 255 + 0.5)     (imageops.py:32-36)

``q`` is monotone non-decreasing in ``x``, so it is fully described by 255
thresholds ``thr[k] = min{x : q(x) >= k}``.  They are found here by bisection
over the ordered bit patterns of non-negative doubles, evaluating ``q`` with
the HOST numpy — the very ``np.power`` the reference runs (SIMD/SVML or libm,
whatever this numpy dispatches to).  The GPU then only needs exact IEEE
arithmetic to form ``x`` and a 255-entry search to produce the reference's
byte, with no pow on the device: bit-exact by construction.  The table is a
per-gamma constant (computed once, cached, uploaded once per device).

This is host-side parameter preparation, not a CPU fallback: no pixel data
ever passes through it.
"""

from __future__ import annotations

import threading

import numpy as np

_LOCK = threading.Lock()
_HOST_CACHE: dict[float, np.ndarray] = {}
_DEV_CACHE: dict[tuple, object] = {}


def quantize_chain(x, gamma):
    """q(x) exactly as the reference evaluates it (recover.py:51-54, imageops.py:32-36)."""
    x = np.asarray(x, dtype=np.float64)
    if gamma == 1.0:
        y = x.copy()
    else:
        y = np.power(x, 1.0 / gamma)
        np.clip(y, 0.0, 1.0, out=y)
    out = np.clip(y, 0.0, 1.0)
    out *= 255.0
    out += 0.5
    np.floor(out, out=out)
    return out.astype(np.uint8)


def compute_thresholds(gamma):
    """Return float64[256]: thr[0] = -1 (unused), thr[k] = smallest x in [0, 1] with q(x) >= k."""
    gamma = float(gamma)
    with _LOCK:
        hit = _HOST_CACHE.get(gamma)
        if hit is not None:
            return hit
    k = np.arange(1, 256, dtype=np.int64)
    lo = np.zeros(255, dtype=np.int64)                         # bits of 0.0  (q(0) = 0 < k)
    hi = np.full(255, np.float64(1.0).view(np.int64))          # bits of 1.0  (q(1) = 255 >= k)
    # invariant: q(lo) < k <= q(hi)
    while True:
        open_ = hi - lo > 1
        if not open_.any():
            break
        mid = lo + (hi - lo) // 2
        qm = quantize_chain(mid.view(np.float64), gamma).astype(np.int64)
        up = qm >= k
        hi = np.where(open_ & up, mid, hi)
        lo = np.where(open_ & ~up, mid, lo)
    thr = hi.view(np.float64)
    # Pin the table: the chain must step exactly at each threshold.
    q_at = quantize_chain(thr, gamma).astype(np.int64)
    q_below = quantize_chain(lo.view(np.float64), gamma).astype(np.int64)
    if not (np.all(q_at >= k) and np.all(q_below < k) and np.all(np.diff(thr) >= 0)):
        raise RuntimeError(f"quantisation chain is not monotone for gamma={gamma}")
    table = np.empty(256, dtype=np.float64)
    table[0] = -1.0
    table[1:] = thr
    table.setflags(write=False)
    with _LOCK:
        _HOST_CACHE[gamma] = table
    return table


def device_thresholds(gamma, device):
    """The threshold table as a float64 CUDA tensor (cached per (gamma, device))."""
    import torch

    dev = torch.device(device)
    key = (float(gamma), dev.index if dev.index is not None else torch.cuda.current_device())
    with _LOCK:
        hit = _DEV_CACHE.get(key)
    if hit is not None:
        return hit
    t = torch.from_numpy(np.array(compute_thresholds(gamma))).to(device=dev)
    with _LOCK:
        _DEV_CACHE[key] = t
    return t
