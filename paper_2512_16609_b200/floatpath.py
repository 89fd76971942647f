"""float64 device path: the reference's stage functions on float64 arrays, and the
float pipeline for frames that need the bilinear resize or the guided filter.

Everything computes on the GPU through libdehaze_b200.so (csrc/floatops.cu);
numpy arrays are copied to the device and results copied back, CUDA tensors
stay on the device.  Argument contracts and error messages follow the
reference's validation.py; the finiteness / range scans run on the device.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native
from .quant import device_thresholds
from .validation import (
    check_float_image_shape,
    check_same_shape,
    check_scalar_map_shape,
    check_stats,
)

F64 = torch.float64


def _lib():
    return _native.lib()


def _dev():
    _lib()
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _call(name, *args):
    rc = getattr(_lib(), name)(*args)
    _native.check(rc, name)


def to_device_f64(x, device=None):
    """Any array-like / tensor -> contiguous float64 CUDA tensor (copy for host input)."""
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if not t.is_cuda:
            t = t.to(device or _dev())
        return t.to(F64).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(device or _dev())


def stats(t):
    """(all finite, min, max) of a CUDA float64 tensor, reduced on the device."""
    n = t.numel()
    out = torch.empty(3, dtype=F64, device=t.device)
    ws = torch.empty(3 * 1024, dtype=F64, device=t.device)
    _call("dhz_f64_stats", t.data_ptr(), n, out.data_ptr(), ws.data_ptr(), _stream())
    ok, lo, hi = out.tolist()
    return ok == 1.0, lo, hi


def check_float_image(x, name="image", clip=False):
    """validation.py:32-56 on the device: returns a float64 CUDA tensor (H, W, 3)."""
    t = to_device_f64(x)
    check_float_image_shape(tuple(t.shape), name)
    ok, lo, hi = stats(t)
    check_stats(name, ok, lo, hi, clip)
    if lo < 0.0 or hi > 1.0:
        t = t.clamp(0.0, 1.0)
    return t


def check_scalar_map(x, name="map"):
    """validation.py:59-72 on the device: returns a float64 CUDA tensor (H, W)."""
    t = to_device_f64(x)
    check_scalar_map_shape(tuple(t.shape), name)
    ok, lo, hi = stats(t)
    check_stats(name, ok, lo, hi, clip=True)  # maps: finiteness only
    return t


def airlight_tensor(a, device):
    from .validation import check_airlight

    return torch.from_numpy(check_airlight(a).copy()).to(device)


# ------------------------------------------------------------------ stages ----
def u8_to_float(frame_t):
    out = torch.empty(frame_t.shape, dtype=F64, device=frame_t.device)
    _call("dhz_u8_to_f64", frame_t.data_ptr(), frame_t.numel(), out.data_ptr(), _stream())
    return out


def float_to_u8(img_t):
    out = torch.empty(img_t.shape, dtype=torch.uint8, device=img_t.device)
    _call("dhz_f64_to_u8", img_t.data_ptr(), img_t.numel(), out.data_ptr(), _stream())
    return out


def to_grayscale(img_t):
    h, w = img_t.shape[:2]
    out = torch.empty((h, w), dtype=F64, device=img_t.device)
    _call("dhz_to_grayscale_f64", img_t.data_ptr(), h * w, out.data_ptr(), _stream())
    return out


def channel_min(img_t):
    h, w = img_t.shape[:2]
    out = torch.empty((h, w), dtype=F64, device=img_t.device)
    _call("dhz_channel_min_f64", img_t.data_ptr(), h * w, out.data_ptr(), _stream())
    return out


def resize_bilinear(img_t, width, height):
    h, w = img_t.shape[:2]
    if (width, height) == (w, h):
        return img_t.clone()
    out = torch.empty((height, width, 3), dtype=F64, device=img_t.device)
    if img_t.dtype == torch.uint8:
        _call("dhz_resize_bilinear_u8", img_t.data_ptr(), h, w, height, width, out.data_ptr(), _stream())
    else:
        _call("dhz_resize_bilinear_f64", img_t.data_ptr(), h, w, height, width, out.data_ptr(), _stream())
    return out


def min_filter(m_t, radius):
    if radius == 0:
        return m_t.clone()
    h, w = m_t.shape
    out = torch.empty_like(m_t)
    tmp = torch.empty_like(m_t)
    _call("dhz_min_filter_f64", m_t.data_ptr(), h, w, int(radius), out.data_ptr(), tmp.data_ptr(), _stream())
    return out


def box_filter(m_t, radius):
    if radius == 0:
        return m_t.clone()
    h, w = m_t.shape
    out = torch.empty_like(m_t)
    tmp = torch.empty_like(m_t)
    _call("dhz_box_filter_f64", m_t.data_ptr(), h, w, int(radius), out.data_ptr(), tmp.data_ptr(), _stream())
    return out


def min_filter_naive(m_t, radius):
    if radius == 0:
        return m_t.clone()
    h, w = m_t.shape
    out = torch.empty_like(m_t)
    _call("dhz_min_filter_naive_f64", m_t.data_ptr(), h, w, int(radius), out.data_ptr(), _stream())
    return out


def box_filter_naive(m_t, radius):
    if radius == 0:
        return m_t.clone()
    h, w = m_t.shape
    out = torch.empty_like(m_t)
    _call("dhz_box_filter_naive_f64", m_t.data_ptr(), h, w, int(radius), out.data_ptr(), _stream())
    return out


def guided_filter(p_t, g_t, radius, eps, floor_t=0.0):
    h, w = p_t.shape
    out = torch.empty_like(p_t)
    ws = torch.empty(7 * h * w, dtype=F64, device=p_t.device)
    _call("dhz_guided_filter_f64", p_t.data_ptr(), g_t.data_ptr(), h, w, int(radius), float(eps), float(floor_t),
          out.data_ptr(), ws.data_ptr(), _stream())
    return out


def transmission(cmin_t, a_t, omega, t_min):
    out = torch.empty_like(cmin_t)
    _call("dhz_transmission_f64", cmin_t.data_ptr(), cmin_t.numel(), a_t.data_ptr(), float(omega),
          float(t_min), out.data_ptr(), _stream())
    return out


def recover(img_t, a_t, t_t):
    out = torch.empty_like(img_t)
    h, w = img_t.shape[:2]
    _call("dhz_recover_f64", img_t.data_ptr(), a_t.data_ptr(), t_t.data_ptr(), h * w, out.data_ptr(), _stream())
    return out


def gamma(img_t, g):
    if g == 1.0:
        return img_t.clone()
    out = torch.empty_like(img_t)
    _call("dhz_gamma_f64", img_t.data_ptr(), img_t.numel(), float(g), out.data_ptr(), _stream())
    return out


def gray_world(img_t):
    out = torch.empty_like(img_t)
    h, w = img_t.shape[:2]
    ws = torch.empty(3 * 256 + 8, dtype=F64, device=img_t.device)
    _call("dhz_gray_world_f64", img_t.data_ptr(), h * w, out.data_ptr(), ws.data_ptr(), _stream())
    return out


def airlight(img_t, dark_t, top_fraction, alpha, return_selection=False):
    npx = dark_t.numel()
    k = max(1, math.floor(top_fraction * npx))
    a = torch.empty(3, dtype=F64, device=img_t.device)
    sel = torch.empty(k, dtype=torch.int32, device=img_t.device)
    _call("dhz_airlight_f64", img_t.data_ptr(), dark_t.data_ptr(), npx, k, float(alpha), a.data_ptr(),
          sel.data_ptr(), _stream())
    return (a, sel) if return_selection else a


def recover_quant(img_t, a_t, t_t, gamma_value):
    h, w = img_t.shape[:2]
    out = torch.empty((h, w, 3), dtype=torch.uint8, device=img_t.device)
    thr = device_thresholds(gamma_value, img_t.device)
    _call("dhz_recover_quant_f64", img_t.data_ptr(), a_t.data_ptr(), t_t.data_ptr(), h * w, thr.data_ptr(),
          out.data_ptr(), _stream())
    return out


# ---------------------------------------------------------------- pipeline ----
def dehaze_float_frame(frame_t, params, telemetry=None):
    """pipeline.py:163-216 with float64 intermediates on the device.

    frame_t: (H, W, 3) uint8 CUDA tensor.  Returns (out uint8 tensor, airlight (3,)
    tensor, maps dict with float64 numpy dark / transmission_coarse / transmission
    when telemetry.capture_maps).
    """
    tel = telemetry
    timers = []

    def mark(name):
        if tel is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            timers.append((name, ev))

    mark(None)
    h, w = int(frame_t.shape[0]), int(frame_t.shape[1])
    if params.resize_to is not None and tuple(params.resize_to) != (w, h):
        rw, rh = (int(v) for v in params.resize_to)
        img = resize_bilinear(frame_t, rw, rh)
    else:
        img = u8_to_float(frame_t)
    mark("resize")
    cmin = channel_min(img)
    mark("channel_min")
    dark = min_filter(cmin, int(params.patch_radius))
    mark("min_filter")
    a = airlight(img, dark, params.top_fraction, params.alpha)
    mark("airlight")
    t_coarse = transmission(cmin, a, params.omega, params.t_min)
    mark("transmission")
    t = t_coarse
    if params.mode == "image":
        t = guided_filter(t_coarse, to_grayscale(img), params.guided_radius, params.guided_eps, params.t_min)
        mark("guided_filter")
    if params.balance_enabled():
        x = recover(img, a, t)
        mark("recover")
        x = gray_world(gamma(x, params.gamma))
        mark("postprocess")
        out = float_to_u8(x)
        mark("output")
    else:
        out = recover_quant(img, a, t, params.gamma)  # recover + gamma + output fused (exact)
        mark("recover")
        mark("postprocess")
        mark("output")
    maps = None
    if tel is not None:
        timers[-1][1].synchronize()
        for (_, e0), (name, e1) in zip(timers, timers[1:]):
            tel.add_time(name, e0.elapsed_time(e1) / 1000.0)
        if tel.capture_maps:
            maps = {"dark": dark.cpu().numpy(), "transmission_coarse": t_coarse.cpu().numpy(),
                    "transmission": t.cpu().numpy()}
    return out, a, maps


def maps_from_native(frame_t, native_maps, a_t, params):
    """capture_maps for the fused u8 path: dark = u8/255 (exact), t from the channel minimum."""
    # true division by 255 (torch's tensor / scalar multiplies by a rounded reciprocal)
    dark = u8_to_float(native_maps["dark_u8"][0].contiguous())
    img = u8_to_float(frame_t)
    t = transmission(channel_min(img), a_t, params.omega, params.t_min)
    tc = t.cpu().numpy()
    return {"dark": dark.cpu().numpy(), "transmission_coarse": tc, "transmission": tc.copy()}


def check_same(a_t, b_t, name_a, name_b):
    check_same_shape(tuple(a_t.shape), tuple(b_t.shape), name_a, name_b)
