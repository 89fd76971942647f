"""Parity of the fused u8 frame pipeline (CUDA) against the CPU oracle.

Bars (BASELINE north_star): dark map and selected top-K set bit-exact; the
airlight, which the device sums in the reference's sequential order, is
required bit-exact too; output frame max |diff| <= 1 LSB with the mismatch
count asserted to be zero (the LUT path reproduces the reference byte for byte).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(frames_np, params):
    from paper_2512_16609_b200.engine import engine_for

    dev = torch.device("cuda", 0)
    batch = torch.from_numpy(np.ascontiguousarray(frames_np)).to(dev)
    out, air, maps = engine_for(dev).run(batch, params, keep_maps=True)
    torch.cuda.synchronize()
    return out.cpu().numpy(), air.cpu().numpy(), maps["dark_u8"].cpu().numpy(), maps["selected"].cpu().numpy()


def _check(frames_np, params, oracle, lsb_mismatch_allowed=0):
    out, air, dark, sel = _run(frames_np, params)
    for i, f in enumerate(frames_np):
        m = {}
        want = oracle.dehaze_frame(f, params, m)
        img = oracle.u8_to_float(f)
        # dark map: bit-exact on the 1/255 grid
        assert np.array_equal(dark[i].astype(np.float64) / 255.0, m["dark"]), f"dark map differs (frame {i})"
        # selected set, in summation order
        want_sel = oracle.select_airlight_pixels(m["dark"], params.top_fraction)
        assert np.array_equal(sel[i].astype(np.int64), want_sel), f"selection differs (frame {i})"
        # airlight: bit-exact
        assert np.array_equal(air[i], m["airlight"]), (air[i], m["airlight"])
        assert np.abs(air[i] - oracle.estimate_airlight(img, m["dark"], params.top_fraction, params.alpha)).max() <= 1e-12
        diff = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        assert diff.max() <= 1
        assert int((diff > 0).sum()) <= lsb_mismatch_allowed, f"{int((diff > 0).sum())} samples differ"


def _params(**kw):
    from paper_2512_16609_b200 import DehazeParams

    kw.setdefault("resize_to", None)
    return DehazeParams(**kw)


def test_synthetic_c3_small(oracle):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=3, width=320, height=180).numpy()
    _check(frames, _params(), oracle)


def test_synthetic_vga_c1(oracle):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c1").numpy()
    _check(frames, _params(), oracle)


@pytest.mark.parametrize("r", [1, 2, 3, 7, 11, 15, 20])
def test_radii(oracle, r):
    rng = np.random.default_rng(100 + r)
    frames = rng.integers(0, 256, size=(2, 72, 96, 3), dtype=np.uint8)
    _check(frames, _params(patch_radius=r), oracle)


@pytest.mark.parametrize("shape", [(37, 53), (24, 30), (1, 1), (1, 17), (17, 1), (5, 300)])
def test_odd_shapes(oracle, shape):
    rng = np.random.default_rng(7)
    frames = rng.integers(0, 256, size=(2,) + shape + (3,), dtype=np.uint8)
    _check(frames, _params(), oracle)


def test_black_and_white(oracle):
    frames = np.stack([np.zeros((24, 32, 3), np.uint8), np.full((24, 32, 3), 255, np.uint8)])
    _check(frames, _params(), oracle)


def test_full_histogram_fallback(oracle):
    # top 50% spans far more than 16 dark levels -> K2b path
    y, x = np.mgrid[0:64, 0:80]
    v = ((x * 3 + y * 2) % 256).astype(np.uint8)
    frames = np.stack([np.stack([v, v, v], -1)] * 2)
    _check(frames, _params(patch_radius=1, top_fraction=0.5), oracle)


def test_top_fraction_one_all_pixels(oracle):
    rng = np.random.default_rng(9)
    frames = rng.integers(0, 256, size=(2, 16, 32, 3), dtype=np.uint8)
    _check(frames, _params(top_fraction=1.0, alpha=1.0), oracle)


@pytest.mark.parametrize("gamma", [1.0, 2.0, 0.7])
def test_gamma_alpha_omega(oracle, gamma):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=1, width=160, height=96).numpy()
    _check(frames, _params(gamma=gamma, alpha=1.0, omega=1.0, t_min=0.1), oracle)


@pytest.mark.parametrize("gamma", [1.2, 1.0])
def test_balance_native(oracle, gamma):
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c4", frames=3, width=192, height=128).numpy()
    p = _params(white_balance=True, gamma=gamma)
    out, air, dark, sel = _run(frames, p)
    for i, f in enumerate(frames):
        m = {}
        want = oracle.dehaze_frame(f, p, m)
        assert np.array_equal(air[i], m["airlight"])
        d = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        assert d.max() <= 1 and int((d > 0).sum()) <= 2


def test_balance_degenerate_black(oracle):
    frames = np.zeros((2, 16, 32, 3), np.uint8)
    p = _params(white_balance=True)
    out, air, _, _ = _run(frames, p)
    for i, f in enumerate(frames):
        assert np.array_equal(out[i], oracle.dehaze_frame(f, p))


@pytest.mark.parametrize("shape", [(37, 53), (24, 30)])
def test_balance_odd_shapes_scalar_path(oracle, shape):
    # widths that are not a multiple of 16 take the scalar balance-sum and K6 kernels
    rng = np.random.default_rng(29)
    frames = rng.integers(0, 256, size=(2,) + shape + (3,), dtype=np.uint8)
    p = _params(white_balance=True)
    out, air, _, _ = _run(frames, p)
    for i, f in enumerate(frames):
        m = {}
        want = oracle.dehaze_frame(f, p, m)
        assert np.array_equal(air[i], m["airlight"])
        d = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        assert d.max() <= 1 and int((d > 0).sum()) <= 2


def test_batches_beyond_the_grid_limit(oracle):
    # more frames than one launch takes (65535): the engine splits the batch
    from paper_2512_16609_b200 import dehaze_batch

    rng = np.random.default_rng(31)
    n = 70000
    frames = rng.integers(0, 256, size=(n, 2, 3, 3), dtype=np.uint8)
    p = _params()
    out, air = dehaze_batch(torch.from_numpy(frames).cuda(), p)
    out, air = out.cpu().numpy(), air.cpu().numpy()
    for i in (0, 65534, 65535, n - 1):
        m = {}
        want = oracle.dehaze_frame(frames[i], p, m)
        assert np.array_equal(out[i], want) and np.array_equal(air[i], m["airlight"])


@pytest.mark.parametrize("bh,direct", [(64, "0"), (16, "1")])
@pytest.mark.parametrize("r", list(range(1, 17)))
def test_k1_tiles_every_radius(oracle, r, bh, direct, monkeypatch):
    """K1's vectorised path (width % 16 == 0, r <= 16) across tile seams: 130 rows
    (three 64-row tile rows, the last partial), 976 columns (three 480-column tiles,
    the last partial); plateaus, extreme values and noise so every lane of the
    16-bit pairs sees 0, 255 and ties.  Both tile heights (64 rows: large batches;
    16 rows: the small-batch launch, nine tile rows here) and both K6 forms (table in
    shared memory; direct gathers for small batches) are forced in turn."""
    monkeypatch.setenv("DHZ_K1_BH", str(bh))
    monkeypatch.setenv("DHZ_K6_DIRECT", direct)
    rng = np.random.default_rng(500 + r)
    H, W = 130, 976
    f0 = rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
    f1 = np.full((H, W, 3), 200, dtype=np.uint8)
    f1[40:90, 470:500] = 255  # plateau across a tile seam
    f1[::7, ::11] = 0        # isolated minima
    f1[:, 959:] = rng.integers(0, 256, size=(H, W - 959, 3), dtype=np.uint8)
    f2 = (np.add.outer(np.arange(H), np.arange(W)) % 256).astype(np.uint8)[..., None].repeat(3, axis=2)
    f2[..., 1] = 255 - f2[..., 1]
    _check(np.stack([f0, f1, f2]), _params(patch_radius=r), oracle)


@pytest.mark.parametrize("r", [1, 4, 7, 8])
def test_k1_tma_variant(oracle, r, monkeypatch):
    """DHZ_K1_TMA=1: K1 with its rows staged by cp.async.bulk.tensor (one stage and one
    mbarrier per warp) instead of LDG.128: same geometry cases as the tile test (partial
    tiles on both axes, so rows and columns outside the frame arrive as TMA zero fill and
    must read as the all-ones neutral), against the oracle and bit-identical to the default."""
    rng = np.random.default_rng(900 + r)
    H, W = 130, 976
    f0 = rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
    f1 = np.full((H, W, 3), 200, dtype=np.uint8)
    f1[::7, ::11] = 0
    f1[:3] = 255
    f1[-2:, -20:] = 1
    frames = np.stack([f0, f1])
    base = _run(frames, _params(patch_radius=r))
    monkeypatch.setenv("DHZ_K1_TMA", "1")
    tma = _run(frames, _params(patch_radius=r))
    for a, b in zip(base, tma):
        assert np.array_equal(a, b)
    _check(frames, _params(patch_radius=r), oracle)
    one = _run(frames[:1, :40, :32], _params(patch_radius=r))  # a single small frame (frame pitch = its size)
    monkeypatch.delenv("DHZ_K1_TMA")
    ref = _run(frames[:1, :40, :32], _params(patch_radius=r))
    for a, b in zip(ref, one):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("shape", [(5, 130, 976), (2, 720, 1280), (1, 16, 16)])
def test_k6_ring_variant(oracle, shape, monkeypatch):
    """DHZ_K6_RING=1: K6 with the frame bytes staged by cp.async.bulk into a two-stage
    shared-memory ring (mbarrier full/empty pairs): several frames per CTA, blocks that
    end inside a stage, a single 16-unit frame; bytes identical to the LDG form and to
    the direct-gather form, and checked against the oracle."""
    n, H, W = shape
    rng = np.random.default_rng(4100 + n)
    frames = rng.integers(0, 256, size=(n, H, W, 3), dtype=np.uint8)
    frames[0, : H // 2] = np.clip(frames[0, : H // 2].astype(np.int16) // 4 + 150, 0, 255).astype(np.uint8)
    p = _params()
    monkeypatch.setenv("DHZ_K6_DIRECT", "0")
    base = _run(frames, p)
    monkeypatch.setenv("DHZ_K6_RING", "1")
    ring = _run(frames, p)
    monkeypatch.setenv("DHZ_K6_DIRECT", "1")
    direct = _run(frames, p)
    for a, b, c in zip(base, ring, direct):
        assert np.array_equal(a, b) and np.array_equal(a, c)
    monkeypatch.setenv("DHZ_K6_DIRECT", "0")
    if n * H * W <= 2_000_000:
        _check(frames, p, oracle)


def test_balance_out_of_band_samples(oracle):
    # uniform noise: most non-minimum samples lie >= 64 levels above their pixel's
    # minimum, outside the banded table (k_balance_band's per-unit correction path)
    rng = np.random.default_rng(37)
    frames = rng.integers(0, 256, size=(3, 64, 96, 3), dtype=np.uint8)
    frames[1, :, :, 0] = 255                      # one saturated channel: d = 255 - m everywhere
    p = _params(white_balance=True)
    out, air, _, _ = _run(frames, p)
    for i, f in enumerate(frames):
        m = {}
        want = oracle.dehaze_frame(f, p, m)
        assert np.array_equal(air[i], m["airlight"])
        d = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        assert d.max() <= 1 and int((d > 0).sum()) <= 2


def test_balance_sums_independent_of_kernel_and_batch():
    # the channel sums are exact integer sums of the quantised g samples, so the
    # banded kernel (16-byte aligned frames), the scalar kernel (a frame buffer one
    # byte off alignment) and any batch composition give the same bytes
    from paper_2512_16609_b200.engine import engine_for
    from paper_2512_16609_b200.synthetic import make_frames

    dev = torch.device("cuda", 0)
    frames = make_frames("c4", frames=3, width=160, height=96).to(dev)
    frames[2] = torch.randint(0, 256, frames[2].shape, dtype=torch.uint8, device=dev, generator=torch.Generator(dev).manual_seed(41))
    p = _params(white_balance=True)
    eng = engine_for(dev)
    aligned, _ = eng.run(frames, p)[:2]
    raw = torch.empty(frames.numel() + 16, dtype=torch.uint8, device=dev)
    shifted = raw[1:1 + frames.numel()].view(frames.shape)
    shifted.copy_(frames)
    assert shifted.data_ptr() % 16 == 1
    scalar, _ = eng.run(shifted, p)[:2]
    single, _ = eng.run(frames[1:2].clone(), p)[:2]
    torch.cuda.synchronize()
    assert torch.equal(aligned, scalar)
    assert torch.equal(aligned[1:2], single)
