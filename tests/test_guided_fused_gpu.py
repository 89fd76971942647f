"""The exact-integer guided filter (guided_fused.cu) in both of its forms: one pass
(DHZ_GUIDED_PATH=fused) and two passes (DHZ_GUIDED_PATH=twopass, pass 1 writing the
fixed-point a, b), which must give the same bytes.

Its box sums are exact integers, so its output must not depend on how the frame is
cut into strips, segments and persistent CTAs (batch size, frame count): checked by
batch invariance.  Against the oracle the bars are the image-mode ones (airlight
bit-exact, <= 1 LSB, <= 2 differing samples per frame); against the strip path the
bytes agree wherever both sit away from a quantisation boundary.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["fused", "twopass"])
def fused_path(monkeypatch, request):
    monkeypatch.setenv("DHZ_GUIDED_PATH", request.param)
    yield request.param


def _params(**kw):
    from paper_2512_16609_b200 import DehazeParams

    return DehazeParams.for_image(**kw)


def _vs_oracle(frames, params, oracle):
    from paper_2512_16609_b200 import dehaze_batch

    out, air = dehaze_batch(frames.cuda(), params)
    out, air = out.cpu().numpy(), air.cpu().numpy()
    for i in range(frames.shape[0]):
        m = {}
        want = oracle.dehaze_frame(frames[i].numpy(), params, m)
        assert np.array_equal(air[i], m["airlight"])
        d = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        assert d.max() <= 1 and int((d > 0).sum()) <= 2, (i, int(d.max()), int((d > 0).sum()))


@pytest.mark.parametrize("balance", [True, False])
@pytest.mark.parametrize("radius", [1, 2, 3, 30, 60, 63])
def test_radii_vs_oracle(oracle, balance, radius):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c5", frames=1, width=1283, height=97)
    _vs_oracle(frames, _params(guided_radius=radius, white_balance=balance), oracle)


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (9, 1), (2, 3), (130, 5), (5, 130), (64, 4100)])
def test_small_and_thin(oracle, shape):
    rng = np.random.default_rng(7)
    frames = torch.from_numpy(rng.integers(0, 256, size=(2,) + shape + (3,), dtype=np.uint8))
    _vs_oracle(frames, _params(guided_radius=9), oracle)


def test_clipped_coarse_t(oracle):
    """omega = 1 makes 1 - (m/255)/max(A) reach t_min: the clipped-p sums are used."""
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c2", frames=2, width=517, height=211)
    _vs_oracle(frames, _params(omega=1.0, t_min=0.3, guided_radius=20), oracle)
    _vs_oracle(frames, _params(omega=1.0, t_min=0.3, guided_radius=20, white_balance=False), oracle)


def test_batch_invariance_exact():
    """Exact sums: a frame's bytes are the same alone, in a pair, or in a large batch
    (where the persistent CTAs cut the columns at different rows)."""
    from paper_2512_16609_b200 import dehaze_batch
    from paper_2512_16609_b200.synthetic import make_frames

    p = _params(patch_radius=15, guided_radius=60)
    frames = make_frames("c5", frames=12, width=2048, height=1100, device="cuda")
    out, air = dehaze_batch(frames, p)
    for lo, hi in [(0, 1), (5, 7), (11, 12)]:
        o, a = dehaze_batch(frames[lo:hi].clone(), p)
        assert torch.equal(o, out[lo:hi]) and torch.equal(a, air[lo:hi])


def test_matches_strip_path(monkeypatch):
    from paper_2512_16609_b200 import dehaze_batch
    from paper_2512_16609_b200.synthetic import make_frames

    p = _params(patch_radius=15, guided_radius=60)
    frames = make_frames("c5", frames=2, width=4096, height=512, device="cuda")
    out_f, air_f = dehaze_batch(frames, p)
    monkeypatch.setenv("DHZ_GUIDED_PATH", "strip")
    out_s, air_s = dehaze_batch(frames, p)
    assert torch.equal(air_f, air_s)
    d = (out_f.to(torch.int16) - out_s.to(torch.int16)).abs()
    assert int(d.max()) <= 1 and int((d > 0).sum()) <= 4


@pytest.mark.parametrize("balance", [True, False])
def test_two_forms_identical(monkeypatch, balance):
    """One pass and two passes compute the same integers and the same fp64 code."""
    from paper_2512_16609_b200 import dehaze_batch
    from paper_2512_16609_b200.synthetic import make_frames

    p = _params(patch_radius=15, guided_radius=60, white_balance=balance)
    frames = make_frames("c5", frames=3, width=4100, height=700, device="cuda")
    outs = {}
    for path in ("fused", "twopass"):
        monkeypatch.setenv("DHZ_GUIDED_PATH", path)
        outs[path] = dehaze_batch(frames, p)
    assert torch.equal(outs["fused"][0], outs["twopass"][0])
    assert torch.equal(outs["fused"][1], outs["twopass"][1])
