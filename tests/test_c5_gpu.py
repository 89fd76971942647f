"""Image-mode parity at the BASELINE C5 geometry (frames at least 4096 wide).

C5 is 64 x 7680x4320 in image mode with a 31x31 dark-channel patch
(patch_radius=15), guided radius 60, eps 1e-3 and gray-world balance (the image
default).  Frames this wide take the default two-pass exact guided filter (and, for guided
radii above 63 or with DHZ_GUIDED_PATH=strip, the CPT = 4 strip kernels), so they are
compared with the CPU oracle (reference estimation.py:110-172, pipeline.py:163-216)
here, on narrow 4096-wide strips of the C5 generator with balance on and off, and
on one full 7680x4320 C5 frame.

Bars: airlight bit-exact; output max |diff| <= 1 LSB with at most
2 differing samples per frame.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _c5_params(**kw):
    from paper_2512_16609_b200 import DehazeParams

    return DehazeParams.for_image(patch_radius=15, guided_radius=60, guided_eps=1e-3, **kw)


def _compare(frames, params, oracle):
    from paper_2512_16609_b200 import dehaze_batch

    out, air = dehaze_batch(frames.cuda(), params)
    out, air = out.cpu().numpy(), air.cpu().numpy()
    for i in range(frames.shape[0]):
        m = {}
        want = oracle.dehaze_frame(frames[i].numpy(), params, m)
        assert np.array_equal(air[i], m["airlight"]), (i, air[i], m["airlight"])
        d = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        assert d.max() <= 1 and int((d > 0).sum()) <= 2, (i, int(d.max()), int((d > 0).sum()))


@pytest.mark.parametrize("path", ["default", "strip"])
@pytest.mark.parametrize("balance", [True, False])
@pytest.mark.parametrize("width,height", [(4096, 160), (4104, 131)])
def test_wide_strips(oracle, monkeypatch, path, balance, width, height):
    """The default (two-pass exact) filter and the strip kernels (CPT = 4 at this width;
    the default for guided radii above 63)."""
    from paper_2512_16609_b200.synthetic import make_frames

    if path == "strip":
        monkeypatch.setenv("DHZ_GUIDED_PATH", "strip")
    frames = make_frames("c5", frames=2, width=width, height=height)
    _compare(frames, _c5_params(white_balance=balance), oracle)


@pytest.mark.parametrize("radius", [1, 17, 30, 63, 64])
def test_wide_radii(oracle, radius):
    """Radii around the wide-frame kernel's limits (window 3 .. 129 columns)."""
    from paper_2512_16609_b200 import DehazeParams
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c5", frames=1, width=4352, height=96)
    _compare(frames, DehazeParams.for_image(guided_radius=radius, white_balance=radius % 2 == 1), oracle)


def test_c5_full_frame(oracle):
    """One full BASELINE C5 frame (7680x4320): the oracle takes ~10 s and ~6 GB."""
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c5", frames=1, device="cuda").cpu()
    _compare(frames, _c5_params(), oracle)
