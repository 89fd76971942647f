"""CPU oracle for the Hazedefy per-frame dehaze path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(``/root/reference/pkg/src/dehaze``) used as the *checker* for the CUDA
product path.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package (``paper_2512_16609_b200``) never imports it and has no
CPU fallback.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference (in the
survey container, where ``/root/reference`` exists) on seeded inputs and
commits the results as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this restatement against those fixtures bit-for-bit (``-m "not gpu"``),
and against the live reference when it is importable.

Every function cites the reference file:line whose arithmetic it restates.
The floating-point operation ORDER matters for bit-exactness (e.g. a true
division by 255, separate multiply / add without contraction, sequential
row accumulation for means); the comments call out each such choice.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

AIRLIGHT_FLOOR = 1e-6          # estimation.py:33
GRAY_WEIGHTS = (0.299, 0.587, 0.114)  # imageops.py:15
MEAN_FLOOR = 1e-6              # recover.py:20
GAIN_LO, GAIN_HI = 0.5, 2.0    # recover.py:23-24


# --------------------------------------------------------------------------
# conversions (imageops.py)
# --------------------------------------------------------------------------
def u8_to_float(frame):
    """imageops.py:18-21 — float64 true division by 255 (not a reciprocal multiply)."""
    return np.asarray(frame, dtype=np.uint8).astype(np.float64) / 255.0


def float_to_u8(image):
    """imageops.py:24-36 — clip, *255, +0.5, floor, as three separate roundings."""
    x = np.clip(np.asarray(image, dtype=np.float64), 0.0, 1.0)
    x = x * 255.0
    x = x + 0.5
    return np.floor(x).astype(np.uint8)


def to_grayscale(image):
    """imageops.py:39-44 — ((wr*R + wg*G) + wb*B), left-to-right, then clip."""
    wr, wg, wb = GRAY_WEIGHTS
    g = wr * image[:, :, 0] + wg * image[:, :, 1] + wb * image[:, :, 2]
    return np.clip(g, 0.0, 1.0)


def resize_bilinear(image, width, height):
    """imageops.py:47-78 — pixel-centre bilinear, rows first then columns."""
    h, w = image.shape[:2]
    if (width, height) == (w, h):
        return image.copy()
    sx = (np.arange(width, dtype=np.float64) + 0.5) * (w / width) - 0.5
    sy = (np.arange(height, dtype=np.float64) + 0.5) * (h / height) - 0.5
    sx = np.clip(sx, 0.0, w - 1.0)
    sy = np.clip(sy, 0.0, h - 1.0)
    x0 = np.floor(sx).astype(np.intp)
    y0 = np.floor(sy).astype(np.intp)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    fx = (sx - x0)[None, :, None]
    fy = (sy - y0)[:, None, None]
    rows = image[y0] * (1.0 - fy) + image[y1] * fy
    out = rows[:, x0] * (1.0 - fx) + rows[:, x1] * fx
    return np.clip(out, 0.0, 1.0)


# --------------------------------------------------------------------------
# dark channel (estimation.py:35-43, morphology.py:63-92)
# --------------------------------------------------------------------------
def channel_min(image):
    """estimation.py:35-38 — min(min(R, G), B)."""
    return np.minimum(np.minimum(image[:, :, 0], image[:, :, 1]), image[:, :, 2])


def _sliding_min_axis(m, radius, axis):
    # Window [i-r, i+r] clamped to the array: replicate padding never changes
    # a minimum, so clamping the window is identical to morphology.py:21-31.
    n = m.shape[axis]
    out = m.copy()
    for s in range(1, radius + 1):
        if s >= n:
            break
        lo = [slice(None)] * m.ndim
        hi = [slice(None)] * m.ndim
        lo[axis] = slice(0, n - s)
        hi[axis] = slice(s, n)
        # out[i] = min(out[i], m[i+s]) and out[i+s] = min(out[i+s], m[i])
        np.minimum(out[tuple(lo)], m[tuple(hi)], out=out[tuple(lo)])
        np.minimum(out[tuple(hi)], m[tuple(lo)], out=out[tuple(hi)])
    return out


def min_filter(m, radius):
    """morphology.py:63-73 — separable (2r+1)^2 erosion, replicate border.

    min is exact, so any evaluation order gives the reference bits; this
    restatement uses shifted-slice minima instead of van Herk/Gil-Werman.
    """
    m = np.asarray(m, dtype=np.float64)
    if radius == 0:
        return m.copy()
    return _sliding_min_axis(_sliding_min_axis(m, radius, 1), radius, 0)


def min_filter_naive(m, radius):
    """morphology.py:76-92 — per-pixel clamped-window scan (small inputs only)."""
    m = np.asarray(m, dtype=np.float64)
    h, w = m.shape
    out = np.empty_like(m)
    for i in range(h):
        for j in range(w):
            out[i, j] = m[max(0, i - radius):i + radius + 1, max(0, j - radius):j + radius + 1].min()
    return out


def dark_channel(image, radius):
    """estimation.py:41-43."""
    return min_filter(channel_min(image), radius)


# --------------------------------------------------------------------------
# airlight (estimation.py:46-84)
# --------------------------------------------------------------------------
def top_k(n, top_fraction):
    """estimation.py:72 — K = max(1, floor(top_fraction * n)) in Python float arithmetic."""
    return max(1, math.floor(top_fraction * n))


def select_airlight_pixels(dark, top_fraction):
    """estimation.py:71-82 — the ordered selection.

    Returns the flat indices in the order the reference sums them: every
    pixel strictly above the K-th largest value (ascending index), then the
    first ``K - above`` pixels equal to it (ascending index).  When K == n the
    reference takes ``arange(n)``.
    """
    flat = np.asarray(dark, dtype=np.float64).ravel()
    n = flat.size
    k = top_k(n, top_fraction)
    if k >= n:
        return np.arange(n)
    thr = np.sort(flat)[n - k]          # K-th largest == (n-k)-th smallest
    above = np.flatnonzero(flat > thr)
    ties = np.flatnonzero(flat == thr)[: k - above.size]
    return np.concatenate([above, ties])


def estimate_airlight(image, dark, top_fraction, alpha):
    """estimation.py:46-84 — mean RGB at the selection, *alpha, floored at 1e-6.

    The mean over axis 0 of a (K, 3) array is a sequential row accumulation
    in numpy followed by a true division by K; restated explicitly.
    """
    sel = select_airlight_pixels(dark, top_fraction)
    rows = image.reshape(-1, 3)[sel]
    acc = np.zeros(3)
    for r in rows:                      # sequential, selection order
        acc = acc + r
    mean = acc / float(sel.size)
    return np.maximum(alpha * mean, AIRLIGHT_FLOOR)


def estimate_airlight_fast(image, dark, top_fraction, alpha):
    """Same as estimate_airlight; uses numpy's axis-0 mean (sequential rows)."""
    sel = select_airlight_pixels(dark, top_fraction)
    mean = image.reshape(-1, 3)[sel].mean(axis=0)
    return np.maximum(alpha * mean, AIRLIGHT_FLOOR)


# --------------------------------------------------------------------------
# transmission, guided filter (estimation.py:87-172)
# --------------------------------------------------------------------------
def transmission_from_channel_min(cmin, airlight, omega, t_min):
    """estimation.py:100-101 — 1 - omega*(cmin/max(A)), clipped to [t_min, 1]."""
    t = 1.0 - omega * (cmin / np.max(airlight))
    return np.clip(t, t_min, 1.0)


def box_filter(m, radius):
    """estimation.py:110-125 — edge-padded fp64 summed-area table, / k^2."""
    m = np.asarray(m, dtype=np.float64)
    if radius == 0:
        return m.copy()
    k = 2 * radius + 1
    p = np.pad(m, radius, mode="edge")
    sat = np.zeros((p.shape[0] + 1, p.shape[1] + 1))
    sat[1:, 1:] = p.cumsum(axis=0).cumsum(axis=1)
    win = sat[k:, k:] - sat[:-k, k:] - sat[k:, :-k] + sat[:-k, :-k]
    return win / float(k * k)


def guided_filter(p, guide, radius, eps):
    """estimation.py:144-172 — He et al. guided filter on box means, clip [0, 1]."""
    mi = box_filter(guide, radius)
    mp = box_filter(p, radius)
    cip = box_filter(guide * p, radius)
    cii = box_filter(guide * guide, radius)
    var = cii - mi * mi
    cov = cip - mi * mp
    a = cov / (var + eps)
    b = mp - a * mi
    q = box_filter(a, radius) * guide + box_filter(b, radius)
    return np.clip(q, 0.0, 1.0)


# --------------------------------------------------------------------------
# recovery and post-processing (recover.py:28-69)
# --------------------------------------------------------------------------
def recover_radiance(image, airlight, t):
    """recover.py:40-43 — ((I - A) / t) + A, clip [0, 1]; three roundings."""
    out = image - airlight
    out = out / t[:, :, None]
    out = out + airlight
    return np.clip(out, 0.0, 1.0)


def gamma_correct(image, gamma):
    """recover.py:46-54 — identity copy at gamma == 1, else power(x, 1/gamma)."""
    if gamma == 1.0:
        return image.copy()
    return np.clip(np.power(image, 1.0 / gamma), 0.0, 1.0)


def gray_world_balance(image):
    """recover.py:57-69 — per-channel sequential means, gains clipped to [0.5, 2]."""
    means = image.mean(axis=(0, 1))
    if means.min() < MEAN_FLOOR:
        return image.copy()
    gains = np.clip(means.mean() / means, GAIN_LO, GAIN_HI)
    return np.clip(image * gains, 0.0, 1.0)


# --------------------------------------------------------------------------
# pipeline (pipeline.py:163-308)
# --------------------------------------------------------------------------
class OracleParams:
    """Field-for-field stand-in for DehazeParams (pipeline.py:52-114)."""

    def __init__(self, mode="video", patch_radius=7, top_fraction=0.001, alpha=0.8,
                 omega=0.5, t_min=0.05, guided_radius=40, guided_eps=1e-3, gamma=1.2,
                 white_balance=None, resize_to=(640, 480)):
        self.mode = mode
        self.patch_radius = patch_radius
        self.top_fraction = top_fraction
        self.alpha = alpha
        self.omega = omega
        self.t_min = t_min
        self.guided_radius = guided_radius
        self.guided_eps = guided_eps
        self.gamma = gamma
        self.white_balance = white_balance
        self.resize_to = resize_to

    @classmethod
    def of(cls, params):
        if params is None:
            return cls()
        if isinstance(params, cls):
            return params
        return cls(**{k: getattr(params, k) for k in (
            "mode", "patch_radius", "top_fraction", "alpha", "omega", "t_min",
            "guided_radius", "guided_eps", "gamma", "white_balance", "resize_to")})

    def balance_enabled(self):
        if self.white_balance is None:
            return self.mode == "image"
        return bool(self.white_balance)


def dehaze_frame(frame, params=None, maps=None):
    """pipeline.py:163-216 — returns the u8 output; fills ``maps`` if a dict is given.

    ``maps`` receives: dark, transmission_coarse, transmission (float64, as
    FrameTelemetry.record_map keeps them) and airlight (3,).
    """
    p = OracleParams.of(params)
    img = u8_to_float(frame)
    if p.resize_to is not None:
        w, h = p.resize_to
        if (w, h) != (img.shape[1], img.shape[0]):
            img = resize_bilinear(img, w, h)
    cmin = channel_min(img)
    dark = min_filter(cmin, p.patch_radius)
    a = estimate_airlight_fast(img, dark, p.top_fraction, p.alpha)
    t = transmission_from_channel_min(cmin, a, p.omega, p.t_min)
    t_coarse = t
    if p.mode == "image":
        t = guided_filter(t, to_grayscale(img), p.guided_radius, p.guided_eps)
        t = np.maximum(t, p.t_min)
    out = recover_radiance(img, a, t)
    out = gamma_correct(out, p.gamma)
    if p.balance_enabled():
        out = gray_world_balance(out)
    if maps is not None:
        maps["dark"] = dark
        maps["transmission_coarse"] = t_coarse
        maps["transmission"] = t
        maps["airlight"] = a
    return float_to_u8(out)


def dehaze_image(frame, params=None, maps=None):
    """pipeline.py:219-229 — forces image mode."""
    p = OracleParams.of(params) if params is not None else OracleParams(mode="image", resize_to=None)
    if p.mode != "image":
        q = OracleParams.of(p)
        p = OracleParams(**{**q.__dict__, "mode": "image"})
    return dehaze_frame(frame, p, maps)


def process_stream(frames, params=None, workers=1):
    """pipeline.py:232-308 — in-order outputs and airlight trace (no sink/timing).

    workers > 1 fans frames out to a thread pool (numpy releases the GIL),
    which is how the reference reaches its multi-core throughput.
    """
    def one(f):
        m = {}
        out = dehaze_frame(f, params, m)
        return out, m["airlight"]

    frames = list(frames)
    if workers <= 1:
        res = [one(f) for f in frames]
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            res = list(pool.map(one, frames))
    return [r[0] for r in res], [r[1] for r in res]


# --------------------------------------------------------------------------
# quantisation thresholds (used to pin the product's threshold tables)
# --------------------------------------------------------------------------
def quantize_after_gamma(x, gamma):
    """The composite x -> u8 of recover.py:53-54 followed by imageops.py:32-36."""
    x = np.asarray(x, dtype=np.float64)
    y = x.copy() if gamma == 1.0 else np.clip(np.power(x, 1.0 / gamma), 0.0, 1.0)
    return float_to_u8(y)


# --------------------------------------------------------------------------
# opt-in temporal stabilisation (north_star; NOT in the reference: SPEC.md:267
# lists temporal smoothing as a non-goal).  Restated here only to check the
# device recurrence bit for bit: plain Python floats are IEEE doubles with one
# rounding per operation and no fused multiply-add.
# --------------------------------------------------------------------------
def ema_trace(trace, lam, carry=None):
    """A'_f = lam * A'_{f-1} + (1 - lam) * A_f per channel; A'_-1 = carry, else A'_0 = A_0."""
    keep, take = float(lam), 1.0 - float(lam)
    out = []
    prev = None if carry is None else [float(v) for v in carry]
    for row in np.asarray(trace, dtype=np.float64):
        cur = [float(v) for v in row]
        if prev is not None:
            cur = [keep * p + take * c for p, c in zip(prev, cur)]
        out.append(cur)
        prev = cur
    return np.array(out, dtype=np.float64).reshape(-1, 3)


def dehaze_stabilised(frames, params, lam):
    """The stabilised clip: per-frame airlight -> ema_trace -> each frame recovered with A'."""
    p = OracleParams.of(params)
    airs = []
    for f in frames:
        m = {}
        dehaze_frame(f, p, m)
        airs.append(m["airlight"])
    smooth = ema_trace(np.array(airs), lam)
    outs = [dehaze_frame_with_airlight(f, p, a) for f, a in zip(frames, smooth)]
    return outs, smooth


def dehaze_frame_with_airlight(frame, params, airlight):
    """pipeline.py:163-216 with the airlight given instead of estimated."""
    p = OracleParams.of(params)
    img = u8_to_float(frame)
    if p.resize_to is not None:
        w, h = p.resize_to
        if (w, h) != (img.shape[1], img.shape[0]):
            img = resize_bilinear(img, w, h)
    cmin = channel_min(img)
    a = np.asarray(airlight, dtype=np.float64)
    t = transmission_from_channel_min(cmin, a, p.omega, p.t_min)
    if p.mode == "image":
        t = guided_filter(t, to_grayscale(img), p.guided_radius, p.guided_eps)
        t = np.maximum(t, p.t_min)
    out = recover_radiance(img, a, t)
    out = gamma_correct(out, p.gamma)
    if p.balance_enabled():
        out = gray_world_balance(out)
    return float_to_u8(out)
