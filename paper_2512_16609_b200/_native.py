"""ctypes binding of libdehaze_b200.so (include/dehaze_b200.h).

The library is the only compute path of this package: there is no CPU
fallback.  Loading fails loudly when the .so is missing (run
``__graft_entry__.build()`` / ``make -C paper_2512_16609_b200/csrc``) or when
no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdehaze_b200.so")

DHZ_OK = 0
DHZ_E_INVALID = -1
DHZ_E_CUDA = -2
DHZ_E_WORKSPACE = -3
DHZ_E_UNSUPPORTED = -4
ABI_VERSION = 1


class DhzParams(ctypes.Structure):
    """struct dhz_params (include/dehaze_b200.h)."""

    _fields_ = [
        ("mode", ctypes.c_int32),
        ("patch_radius", ctypes.c_int32),
        ("top_k", ctypes.c_int64),
        ("alpha", ctypes.c_double),
        ("omega", ctypes.c_double),
        ("t_min", ctypes.c_double),
        ("guided_radius", ctypes.c_int32),
        ("balance", ctypes.c_int32),
        ("guided_eps", ctypes.c_double),
        ("gamma", ctypes.c_double),
        ("thresholds", ctypes.c_void_p),
    ]


class NativeError(RuntimeError):
    """A libdehaze_b200 call failed (message from dhz_last_error())."""


_c_void_p = ctypes.c_void_p
_c_int = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_size = ctypes.c_size_t
_P = ctypes.POINTER(DhzParams)

# name -> (restype, argtypes); the exported symbol set of include/dehaze_b200.h
SIGNATURES = {
    "dhz_last_error": (ctypes.c_char_p, []),
    "dhz_abi_version": (_c_int, []),
    "dhz_device_count": (_c_int, []),
    "dhz_frames_u8_workspace": (_c_size, [_c_int, _c_int, _c_int, _P]),
    "dhz_frames_u8": (_c_int, [_c_void_p, _c_i64, _c_int, _c_int, _c_int, _P, _c_void_p, _c_i64,
                               _c_void_p, _c_void_p, _c_size, _c_void_p, _c_void_p]),
    "dhz_frames_u8_layout": (_c_int, [_c_int, _c_int, _c_int, _P, ctypes.POINTER(_c_i64)]),
    "dhz_frames_resize_u8_workspace": (_c_size, [_c_int, _c_int, _c_int, _c_int, _c_int, _P]),
    "dhz_frames_resize_u8": (_c_int, [_c_void_p, _c_i64, _c_int, _c_int, _c_int, _c_int, _c_int, _P, _c_void_p,
                                      _c_i64, _c_void_p, _c_void_p, _c_size, _c_void_p, _c_void_p]),
    "dhz_frames_resize_u8_layout": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _P,
                                             ctypes.POINTER(_c_i64)]),
    "dhz_frames_u8_airlight": (_c_int, [_c_void_p, _c_i64, _c_int, _c_int, _c_int, _P, _c_void_p, _c_void_p,
                                        _c_size, _c_void_p]),
    "dhz_frames_u8_recover": (_c_int, [_c_void_p, _c_i64, _c_int, _c_int, _c_int, _P, _c_void_p, _c_void_p,
                                       _c_i64, _c_void_p, _c_size, _c_void_p]),
    "dhz_frames_resize_u8_airlight": (_c_int, [_c_void_p, _c_i64, _c_int, _c_int, _c_int, _c_int, _c_int, _P,
                                               _c_void_p, _c_void_p, _c_size, _c_void_p]),
    "dhz_frames_resize_u8_recover": (_c_int, [_c_void_p, _c_i64, _c_int, _c_int, _c_int, _c_int, _c_int, _P,
                                              _c_void_p, _c_void_p, _c_i64, _c_void_p, _c_size, _c_void_p]),
    # multi-GPU plumbing and the opt-in stabilisation
    "dhz_comm_init": (_c_int, [_c_int, ctypes.POINTER(_c_int), ctypes.POINTER(_c_void_p)]),
    "dhz_comm_destroy": (_c_int, [_c_void_p]),
    "dhz_allgather_airlight": (_c_int, [_c_void_p, ctypes.POINTER(_c_void_p), ctypes.POINTER(_c_int),
                                        ctypes.POINTER(_c_void_p), ctypes.POINTER(_c_void_p)]),
    "dhz_ema_airlight": (_c_int, [_c_void_p, _c_int, ctypes.c_double, _c_void_p, _c_void_p, _c_void_p]),
    # float64 stage operations
    "dhz_f64_stats": (_c_int, [_c_void_p, _c_i64, _c_void_p, _c_void_p, _c_void_p]),
    "dhz_u8_to_f64": (_c_int, [_c_void_p, _c_i64, _c_void_p, _c_void_p]),
    "dhz_f64_to_u8": (_c_int, [_c_void_p, _c_i64, _c_void_p, _c_void_p]),
    "dhz_to_grayscale_f64": (_c_int, [_c_void_p, _c_i64, _c_void_p, _c_void_p]),
    "dhz_resize_bilinear_f64": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_void_p, _c_void_p]),
    "dhz_resize_bilinear_u8": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_void_p, _c_void_p]),
    "dhz_channel_min_f64": (_c_int, [_c_void_p, _c_i64, _c_void_p, _c_void_p]),
    "dhz_min_filter_f64": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_void_p, _c_void_p]),
    "dhz_min_filter_naive_f64": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_void_p]),
    "dhz_box_filter_naive_f64": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_void_p]),
    "dhz_box_filter_f64": (_c_int, [_c_void_p, _c_int, _c_int, _c_int, _c_void_p, _c_void_p, _c_void_p]),
    "dhz_guided_filter_f64": (_c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_int, ctypes.c_double,
                                       ctypes.c_double, _c_void_p, _c_void_p, _c_void_p]),
    "dhz_transmission_f64": (_c_int, [_c_void_p, _c_i64, _c_void_p, ctypes.c_double, ctypes.c_double,
                                      _c_void_p, _c_void_p]),
    "dhz_recover_f64": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_i64, _c_void_p, _c_void_p]),
    "dhz_recover_quant_f64": (_c_int, [_c_void_p, _c_void_p, _c_void_p, _c_i64, _c_void_p, _c_void_p,
                                       _c_void_p]),
    "dhz_gamma_f64": (_c_int, [_c_void_p, _c_i64, ctypes.c_double, _c_void_p, _c_void_p]),
    "dhz_gray_world_f64": (_c_int, [_c_void_p, _c_i64, _c_void_p, _c_void_p, _c_void_p]),
    "dhz_airlight_f64": (_c_int, [_c_void_p, _c_void_p, _c_i64, _c_i64, ctypes.c_double, _c_void_p, _c_void_p,
                                  _c_void_p]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"libdehaze_b200.so not found at {path}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.dhz_abi_version() != ABI_VERSION:
            raise ImportError(f"ABI version mismatch: library {lib.dhz_abi_version()}, expected {ABI_VERSION}")
        _lib = lib
        return lib


def lib():
    """The library, with a CUDA device required (the product path)."""
    L = load_library()
    n = L.dhz_device_count()
    if n < 1:
        raise NativeError(
            "paper_2512_16609_b200 needs a CUDA device (B200, sm_100a); none is visible: "
            + L.dhz_last_error().decode(errors="replace")
        )
    return L


def check(rc: int, what: str):
    if rc != DHZ_OK:
        msg = load_library().dhz_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")
