"""Parity of the batched default-resize video path (resize_u8.cu, dhz_frames_resize_u8)
against the CPU oracle.

Bars: dark map (fp64 after the bilinear resize) and selected set bit-exact; the
airlight, summed in the reference's order, bit-exact; output bytes exact without
gray-world balance (exact thresholds), <= 1 LSB with at most 2 flipped samples per
frame with balance (device pow in the gains).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _params(**kw):
    from paper_2512_16609_b200 import DehazeParams

    return DehazeParams(**kw)


def _check(frames_np, params, oracle, per_frame=0):
    from paper_2512_16609_b200.engine import engine_for
    from paper_2512_16609_b200.pipeline import _native_ok

    n, h, w = frames_np.shape[:3]
    assert _native_ok(params, h, w)
    dev = torch.device("cuda", 0)
    batch = torch.from_numpy(np.ascontiguousarray(frames_np)).to(dev)
    out, air, maps = engine_for(dev).run(batch, params, keep_maps=True)
    out, air = out.cpu().numpy(), air.cpu().numpy()
    dark, sel = maps["dark_f64"].cpu().numpy(), maps["selected"].cpu().numpy()
    for i, f in enumerate(frames_np):
        m = {}
        want = oracle.dehaze_frame(f, params, m)
        assert out[i].shape == want.shape
        assert np.array_equal(dark[i], m["dark"]), f"dark map differs (frame {i})"
        want_sel = oracle.select_airlight_pixels(m["dark"], params.top_fraction)
        assert np.array_equal(sel[i].astype(np.int64), want_sel), f"selection differs (frame {i})"
        assert np.array_equal(air[i], m["airlight"]), (air[i], m["airlight"])
        d = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        assert d.max() <= 1, f"frame {i}: max diff {d.max()}"
        assert int((d > 0).sum()) <= per_frame, f"frame {i}: {int((d > 0).sum())} samples differ"


def test_default_params_downscale(oracle):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=3, width=960, height=540).numpy()
    _check(frames, _params(), oracle)   # DehazeParams(): resize_to=(640, 480)


def test_upscale(oracle):
    rng = np.random.default_rng(3)
    frames = rng.integers(0, 256, size=(2, 60, 90, 3), dtype=np.uint8)
    _check(frames, _params(resize_to=(160, 120)), oracle)


@pytest.mark.parametrize("size", [(20, 15), (1, 1), (7, 33), (33, 7), (64, 64)])
def test_odd_targets(oracle, size):
    rng = np.random.default_rng(17)
    frames = rng.integers(0, 256, size=(2, 45, 61, 3), dtype=np.uint8)
    _check(frames, _params(resize_to=size), oracle)


@pytest.mark.parametrize("r", [1, 3, 7, 15, 32])
def test_radii(oracle, r):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=1, width=400, height=300).numpy()
    _check(frames, _params(resize_to=(200, 150), patch_radius=r), oracle)


@pytest.mark.parametrize("tf", [1.0, 0.5, 0.05])
def test_top_fraction(oracle, tf):
    # 1.0: every pixel in index order; 0.5: more candidates than shared memory holds
    rng = np.random.default_rng(23)
    frames = rng.integers(0, 256, size=(2, 100, 120, 3), dtype=np.uint8)
    _check(frames, _params(resize_to=(96, 80), top_fraction=tf), oracle)


def test_flat_frames_all_ties(oracle):
    frames = np.stack([np.full((50, 70, 3), v, np.uint8) for v in (0, 128, 255)])
    _check(frames, _params(resize_to=(40, 30), top_fraction=0.01), oracle)


@pytest.mark.parametrize("gamma", [1.2, 1.0])
def test_balance(oracle, gamma):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c4", frames=2, width=480, height=270).numpy()
    _check(frames, _params(resize_to=(320, 240), white_balance=True, gamma=gamma), oracle, per_frame=2)


@pytest.mark.parametrize("gamma", [2.0, 0.7])
def test_gammas(oracle, gamma):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=1, width=300, height=200).numpy()
    _check(frames, _params(resize_to=(160, 100), gamma=gamma, alpha=1.0, omega=0.9, t_min=0.1), oracle)


def test_process_stream_default_params(oracle):
    from paper_2512_16609_b200 import process_stream
    from paper_2512_16609_b200.synthetic import make_frames

    frames = list(make_frames("c3", frames=4, width=720, height=400).numpy())
    got = []
    stats = process_stream(frames, None, sink=got.append)
    assert stats.frame_count == 4
    for f, o, a in zip(frames, got, stats.airlight_trace):
        m = {}
        want = oracle.dehaze_frame(f, None, m)
        assert o.shape == (480, 640, 3)
        assert np.array_equal(o, want)
        assert np.array_equal(a, m["airlight"])


def test_host_batch_resize(oracle):
    from paper_2512_16609_b200 import DehazeParams, dehaze_host_batch
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=5, width=500, height=300)
    p = DehazeParams(resize_to=(250, 150))
    out, air = dehaze_host_batch(frames.pin_memory(), p, chunk=2)
    for i in range(5):
        m = {}
        want = oracle.dehaze_frame(frames[i].numpy(), p, m)
        assert np.array_equal(out[i].numpy(), want)
        assert np.array_equal(air[i].numpy(), m["airlight"])
