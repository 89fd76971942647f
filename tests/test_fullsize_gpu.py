"""BASELINE-size batches: properties that do not need the oracle to
run the whole batch, plus oracle spot checks on sampled frames.

* batch invariance: a frame's bytes and airlight do not depend on the batch it is
  processed in (same result alone, in a small batch, in the full batch);
* determinism: two runs of the full batch are bit-identical;
* oracle parity on sampled frames of the full batch (C3: 3 frames, C4: 1 frame).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(frames, params):
    from paper_2512_16609_b200 import dehaze_batch

    out, air = dehaze_batch(frames, params)
    torch.cuda.synchronize()
    return out, air


def _invariance(frames, params, picks):
    out, air = _run(frames, params)
    out2, air2 = _run(frames, params)
    assert torch.equal(out, out2) and torch.equal(air, air2), "full batch not deterministic"
    for i in picks:
        o1, a1 = _run(frames[i:i + 1].clone(), params)
        assert torch.equal(o1[0], out[i]) and torch.equal(a1[0], air[i]), f"frame {i} depends on its batch"
    lo = picks[0]
    o3, a3 = _run(frames[lo:lo + 5].clone(), params)
    assert torch.equal(o3, out[lo:lo + 5]) and torch.equal(a3, air[lo:lo + 5])
    return out, air


def _frames(cfg, n=None, w=None, h=None):
    from paper_2512_16609_b200.synthetic import make_frames

    return make_frames(cfg, frames=n, width=w, height=h, device="cuda")


def test_c3_full_batch(oracle):
    from paper_2512_16609_b200 import DehazeParams

    p = DehazeParams(resize_to=None)
    frames = _frames("c3")                       # 300 x 1920x1080
    out, air = _invariance(frames, p, [0, 137, 299])
    for i in (0, 137, 299):
        m = {}
        want = oracle.dehaze_frame(frames[i].cpu().numpy(), p, m)
        assert np.array_equal(out[i].cpu().numpy(), want)
        assert np.array_equal(air[i].cpu().numpy(), m["airlight"])


def test_c4_full_batch_balance(oracle):
    from paper_2512_16609_b200 import DehazeParams

    p = DehazeParams(resize_to=None, white_balance=True)
    frames = _frames("c4")                       # 120 x 3840x2160, gray-world balance
    out, air = _invariance(frames, p, [3, 119])
    m = {}
    want = oracle.dehaze_frame(frames[119].cpu().numpy(), p, m)
    assert np.array_equal(air[119].cpu().numpy(), m["airlight"])
    d = np.abs(out[119].cpu().numpy().astype(np.int16) - want.astype(np.int16))
    assert d.max() <= 1 and int((d > 0).sum()) <= 2


def test_c5_image_batch_invariance():
    from paper_2512_16609_b200 import DehazeParams

    p = DehazeParams.for_image(patch_radius=15, guided_radius=60, guided_eps=1e-3)
    frames = _frames("c5", n=8)                  # 8 of the 64 8K images
    _invariance(frames, p, [0, 7])


def test_c2_image_full(oracle):
    from paper_2512_16609_b200 import DehazeParams

    p = DehazeParams.for_image(guided_radius=30, guided_eps=1e-3)
    frames = _frames("c2", n=3)                  # 1080p images
    out, air = _invariance(frames, p, [1])
    m = {}
    want = oracle.dehaze_frame(frames[1].cpu().numpy(), p, m)
    assert np.array_equal(air[1].cpu().numpy(), m["airlight"])
    d = np.abs(out[1].cpu().numpy().astype(np.int16) - want.astype(np.int16))
    assert d.max() <= 1 and int((d > 0).sum()) <= 2


def test_default_resize_full_batch(oracle):
    from paper_2512_16609_b200 import DehazeParams

    p = DehazeParams()                            # resize_to=(640, 480)
    frames = _frames("c3")
    out, air = _invariance(frames, p, [5, 250])
    m = {}
    want = oracle.dehaze_frame(frames[250].cpu().numpy(), p, m)
    assert np.array_equal(out[250].cpu().numpy(), want)
    assert np.array_equal(air[250].cpu().numpy(), m["airlight"])
