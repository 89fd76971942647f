"""The C ABI library loads and exports every symbol include/dehaze_b200.h declares (no GPU needed)."""
import ctypes
import os
import re

from paper_2512_16609_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "dehaze_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dhz_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 6
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) <= set(_native.SIGNATURES), set(names) - set(_native.SIGNATURES)


def test_abi_version_and_errors():
    lib = _native.load_library()
    assert lib.dhz_abi_version() == _native.ABI_VERSION
    p = _native.DhzParams()
    # invalid parameters are rejected without touching a device
    assert lib.dhz_frames_u8_workspace(1, 0, 4, ctypes.byref(p)) == 0
    assert b"empty frame" in lib.dhz_last_error()
    p.top_k, p.patch_radius, p.thresholds = 5, 1, None
    assert lib.dhz_frames_u8_workspace(1, 4, 4, ctypes.byref(p)) == 0
    assert b"thresholds" in lib.dhz_last_error()


def test_batch_limit_rejected_without_a_device():
    import ctypes

    from paper_2512_16609_b200 import _native
    from paper_2512_16609_b200.engine import MAX_FRAMES_PER_CALL

    lib = _native.load_library()
    p = _native.DhzParams()
    p.mode, p.patch_radius, p.top_k, p.guided_radius = 0, 7, 1, 40
    p.alpha, p.omega, p.t_min, p.guided_eps, p.gamma = 0.8, 0.5, 0.05, 1e-3, 1.2
    p.thresholds = 1  # any non-NULL pointer: only the argument checks run
    assert lib.dhz_frames_u8_workspace(MAX_FRAMES_PER_CALL, 4, 4, ctypes.byref(p)) > 0
    assert lib.dhz_frames_u8_workspace(MAX_FRAMES_PER_CALL + 1, 4, 4, ctypes.byref(p)) == 0
    assert b"split the batch" in lib.dhz_last_error()
