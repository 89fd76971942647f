"""Public-API contracts of the drop-in on the GPU, in the style of the reference's own
unit tests (pkg/tests/test_{morphology,estimation,recover,imageops,pipeline}.py):
properties, known-answer values, error messages and stream semantics."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dz():
    import paper_2512_16609_b200 as m

    return m


def _rand_frame(rng, h=32, w=40):
    return rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)


class TestMorphology:
    def test_random_maps_vs_oracle(self, dz, oracle):
        rng = np.random.default_rng(10)
        for _ in range(30):
            m = rng.random((int(rng.integers(1, 20)), int(rng.integers(1, 20))))
            r = int(rng.integers(0, 8))
            assert np.array_equal(dz.min_filter(m, r), oracle.min_filter_naive(m, r))

    def test_composition(self, dz):
        rng = np.random.default_rng(13)
        for _ in range(10):
            m = rng.random((int(rng.integers(2, 16)), int(rng.integers(2, 16))))
            r1, r2 = int(rng.integers(0, 4)), int(rng.integers(0, 4))
            assert np.array_equal(dz.min_filter(dz.min_filter(m, r1), r2), dz.min_filter(m, r1 + r2))

    def test_identity_copy_and_errors(self, dz):
        m = np.random.default_rng(12).random((5, 6))
        out = dz.min_filter(m, 0)
        assert np.array_equal(out, m) and out is not m
        with pytest.raises(ValueError, match=">= 0"):
            dz.min_filter(np.zeros((3, 3)), -1)
        with pytest.raises(ValueError, match="integer"):
            dz.min_filter(np.zeros((3, 3)), 1.5)
        with pytest.raises(ValueError, match="2-D"):
            dz.min_filter(np.zeros((3, 3, 3)), 1)
        bad = np.zeros((3, 3))
        bad[1, 1] = np.nan
        with pytest.raises(ValueError, match="finite"):
            dz.min_filter(bad, 1)


class TestEstimation:
    def test_airlight_full_sort_oracle(self, dz):
        rng = np.random.default_rng(24)
        for _ in range(20):
            img = rng.random((16, 16, 3))
            dark = dz.dark_channel(img, int(rng.integers(1, 4)))
            flat = dark.ravel()
            order = sorted(range(flat.size), key=lambda i: (-flat[i], i))[:12]
            want = np.maximum(0.8 * img.reshape(-1, 3)[order].mean(axis=0), 1e-6)
            assert np.allclose(dz.estimate_airlight(img, dark, 0.05, 0.8), want, atol=1e-12)

    def test_ties_by_linear_index(self, dz):
        img = np.zeros((2, 4, 3))
        img[0, 1] = 0.9
        img[1, 0] = 0.5
        img[1, 3] = 0.3
        dark = np.array([[0.0, 0.7, 0.0, 0.0], [0.7, 0.0, 0.0, 0.7]])
        assert np.allclose(dz.estimate_airlight(img, dark, top_fraction=0.25, alpha=1.0), 0.7, atol=1e-12)

    def test_dyadic_scale_exact(self, dz):
        rng = np.random.default_rng(28)
        img = rng.uniform(0.1, 0.9, size=(20, 24, 3))
        base = dz.estimate_airlight(img, dz.dark_channel(img, 3))
        for s in (0.5, 0.25):
            assert np.array_equal(dz.estimate_airlight(img * s, dz.dark_channel(img * s, 3)), base * s)

    def test_black_floor_and_errors(self, dz):
        img = np.zeros((8, 8, 3))
        assert np.allclose(dz.estimate_airlight(img, dz.dark_channel(img, 2)), 1e-6)
        with pytest.raises(ValueError, match="top_fraction"):
            dz.estimate_airlight(np.full((4, 4, 3), 0.5), np.zeros((4, 4)), top_fraction=0.0)
        with pytest.raises(ValueError, match="disagree"):
            dz.estimate_airlight(np.zeros((4, 4, 3)), np.zeros((4, 5)))

    def test_transmission_formula_and_clamp(self, dz):
        rng = np.random.default_rng(30)
        for _ in range(10):
            img = rng.random((9, 11, 3))
            a = rng.uniform(0.3, 1.0, size=3)
            omega, t_min = float(rng.uniform(0.1, 1.0)), float(rng.uniform(0.01, 0.4))
            got = dz.estimate_transmission(img, a, omega, t_min)
            want = np.clip(1.0 - omega * img.min(axis=2) / a.max(), t_min, 1.0)
            assert np.allclose(got, want, atol=1e-12)
        with pytest.raises(ValueError, match="airlight"):
            dz.estimate_transmission(np.full((4, 4, 3), 0.5), (0.0, 0.8, 0.8))

    def test_box_filter(self, dz, oracle):
        rng = np.random.default_rng(33)
        for _ in range(20):
            m = rng.random((int(rng.integers(1, 16)), int(rng.integers(1, 16))))
            r = int(rng.integers(0, 6))
            assert np.abs(dz.box_filter(m, r) - oracle.box_filter(m, r)).max() < 1e-12
        assert np.abs(dz.box_filter(np.full((10, 12), 0.41), 4) - 0.41).max() < 1e-12

    def test_guided_filter(self, dz, oracle):
        rng = np.random.default_rng(35)
        for _ in range(5):
            p, g = rng.random((14, 13)), rng.random((14, 13))
            r, eps = int(rng.integers(1, 4)), float(rng.choice([1e-4, 1e-3, 1e-2]))
            assert np.abs(dz.guided_filter(p, g, r, eps) - oracle.guided_filter(p, g, r, eps)).max() < 1e-9
        q = dz.guided_filter(np.full((12, 12), 0.63), rng.random((12, 12)), 3, 1e-3)
        assert np.abs(q - 0.63).max() < 1e-9
        with pytest.raises(ValueError, match=">= 1"):
            dz.guided_filter(np.zeros((5, 5)), np.zeros((5, 5)), 0, 1e-3)
        with pytest.raises(ValueError, match="eps"):
            dz.guided_filter(np.zeros((5, 5)), np.zeros((5, 5)), 2, 0.0)


class TestRecoverAndImageops:
    def test_recover_identity_and_airlight(self, dz):
        rng = np.random.default_rng(41)
        img = rng.random((8, 8, 3))
        assert np.abs(dz.recover_radiance(img, (0.7, 0.8, 0.9), np.ones((8, 8))) - img).max() < 1e-12
        a = np.array([0.6, 0.7, 0.8])
        flat = np.broadcast_to(a, (6, 6, 3)).copy()
        assert np.array_equal(dz.recover_radiance(flat, a, np.full((6, 6), 0.3)), flat)
        t = np.full((4, 4), 0.5)
        t[2, 2] = 0.0
        with pytest.raises(ValueError, match="positive"):
            dz.recover_radiance(np.full((4, 4, 3), 0.5), (0.8, 0.8, 0.8), t)

    def test_gamma_and_balance(self, dz):
        assert np.abs(dz.gamma_correct(np.full((2, 2, 3), 0.25), 2.0) - 0.5).max() < 1e-12
        img = np.random.default_rng(43).random((4, 4, 3))
        out = dz.gamma_correct(img, 1.0)
        assert np.array_equal(out, img) and out is not img
        cast = np.broadcast_to(np.array([0.2, 0.4, 0.6]), (5, 5, 3)).copy()
        assert np.abs(dz.gray_world_balance(cast) - 0.4).max() < 1e-12
        red = np.broadcast_to(np.array([0.1, 0.4, 0.4]), (5, 5, 3)).copy()
        assert np.allclose(dz.gray_world_balance(red)[0, 0], (0.2, 0.3, 0.3), atol=1e-12)
        black = np.zeros((4, 4, 3))
        assert np.array_equal(dz.gray_world_balance(black), black)

    def test_conversions(self, dz):
        vals = np.arange(256, dtype=np.uint8)
        frame = np.stack([vals, vals, vals], -1)[None]
        assert np.array_equal(dz.float_to_u8(dz.u8_to_float(frame)), frame)
        out = dz.float_to_u8(np.broadcast_to(np.array([0.5, 0.25, 0.75]), (2, 2, 3)).copy())
        assert out[0, 0].tolist() == [128, 64, 191]
        with pytest.raises(ValueError, match="uint8"):
            dz.u8_to_float(np.zeros((4, 4, 3), np.float32))
        with pytest.raises(ValueError, match="finite"):
            dz.float_to_u8(np.full((2, 2, 3), np.nan))
        assert abs(dz.to_grayscale(np.broadcast_to(np.array([1.0, 0, 0]), (2, 2, 3)).copy())[0, 0] - 0.299) < 1e-12

    def test_resize(self, dz, oracle):
        rng = np.random.default_rng(3)
        for _ in range(10):
            h, w = (int(v) for v in rng.integers(1, 12, size=2))
            img = rng.random((h, w, 3))
            ow, oh = (int(v) for v in rng.integers(1, 20, size=2))
            assert np.array_equal(dz.resize_bilinear(img, ow, oh), oracle.resize_bilinear(img, ow, oh))
        with pytest.raises(ValueError, match="positive"):
            dz.resize_bilinear(np.full((2, 2, 3), 0.5), 0, 4)
        with pytest.raises(ValueError, match="outside"):
            dz.resize_bilinear(np.full((2, 2, 3), 1.5), 1, 1)


class TestPipeline:
    def test_default_resize_and_native(self, dz):
        rng = np.random.default_rng(64)
        assert dz.dehaze_frame(_rand_frame(rng, 24, 24)).shape == (480, 640, 3)
        assert dz.dehaze_frame(_rand_frame(rng, 20, 26), dz.DehazeParams(resize_to=None)).shape == (20, 26, 3)
        assert dz.dehaze_image(_rand_frame(rng, 37, 53)).shape == (37, 53, 3)

    def test_stage_sets_and_maps(self, dz):
        rng = np.random.default_rng(66)
        tel = dz.FrameTelemetry()
        for _ in range(3):
            dz.dehaze_frame(_rand_frame(rng), dz.DehazeParams(resize_to=None), tel)
        assert set(tel.counts) == set(dz.VIDEO_STAGES) and all(v == 3 for v in tel.counts.values())
        assert len(tel.airlights) == 3 and all(t >= 0.0 for ts in tel.timings.values() for t in ts)
        tel_i = dz.FrameTelemetry(capture_maps=True)
        dz.dehaze_frame(_rand_frame(rng), dz.DehazeParams.for_image(), tel_i)
        assert set(tel_i.counts) == set(dz.IMAGE_STAGES) and tel_i.counts["guided_filter"] == 1
        assert set(tel_i.maps) == {"dark", "transmission_coarse", "transmission"}
        off = dz.FrameTelemetry()
        dz.dehaze_frame(_rand_frame(rng), dz.DehazeParams(resize_to=None), off)
        assert off.maps == {}

    def test_refinement_smoother_and_floor(self, dz):
        frame = np.random.default_rng(75).integers(0, 256, size=(60, 80, 3), dtype=np.uint8)
        tv, ti = dz.FrameTelemetry(capture_maps=True), dz.FrameTelemetry(capture_maps=True)
        dz.dehaze_frame(frame, dz.DehazeParams(resize_to=None), tv)
        dz.dehaze_frame(frame, dz.DehazeParams.for_image(t_min=0.2), ti)

        def lap(t):
            return np.abs(t[:-2, 1:-1] + t[2:, 1:-1] + t[1:-1, :-2] + t[1:-1, 2:] - 4 * t[1:-1, 1:-1]).mean()

        assert lap(ti.maps["transmission"]) <= lap(tv.maps["transmission"])
        assert ti.maps["transmission"].min() >= 0.2

    def test_white_frame_uniform_and_determinism(self, dz):
        out = dz.dehaze_frame(np.full((24, 30, 3), 255, np.uint8), dz.DehazeParams(resize_to=None))
        assert all(np.unique(out[:, :, c]).size == 1 for c in range(3))
        f = _rand_frame(np.random.default_rng(61))
        p = dz.DehazeParams(resize_to=None)
        assert np.array_equal(dz.dehaze_frame(f, p), dz.dehaze_frame(f, p))
        with pytest.raises(ValueError, match="uint8"):
            dz.dehaze_frame(np.zeros((8, 8, 3)), p)

    def test_stream_order_workers_and_abort(self, dz):
        rng = np.random.default_rng(71)
        frames = [_rand_frame(rng) for _ in range(8)]
        p = dz.DehazeParams(resize_to=None)
        seq, par = [], []
        s1 = dz.process_stream(frames, p, sink=seq.append, workers=1)
        s2 = dz.process_stream(iter(frames), p, sink=par.append, workers=3)
        want = [dz.dehaze_frame(f, p) for f in frames]
        assert all(np.array_equal(a, b) for a, b in zip(seq, want))
        assert all(np.array_equal(a, b) for a, b in zip(seq, par))
        assert all(np.array_equal(a, b) for a, b in zip(s1.airlight_trace, s2.airlight_trace))
        assert s1.frame_count == 8 and abs(s1.fps - s1.frame_count / s1.wall_time) < 1e-9
        got = []
        bad = [_rand_frame(rng, 16, 20), _rand_frame(rng, 16, 20), _rand_frame(rng, 16, 24)]
        with pytest.raises(ValueError, match=r"frame 2.*24x16.*20x16"):
            dz.process_stream(bad, p, sink=got.append)
        assert len(got) == 2
        with pytest.raises(ValueError, match="workers"):
            dz.process_stream([], p, workers=0)
        empty = dz.process_stream([], p)
        assert empty.frame_count == 0 and empty.airlight_trace == []

    def test_stream_outputs_own_their_memory(self, dz, monkeypatch):
        """Fresh outputs are views of their own pinned tensors while the caller-held bytes
        fit the budget, plain arrays past it; the bytes are the same either way, kept
        frames stay intact while later batches run, and dropped frames return the budget."""
        import gc

        from paper_2512_16609_b200 import pipeline as pl
        from paper_2512_16609_b200.synthetic import make_frames

        frames = list(make_frames("c3", frames=40, width=800, height=448).numpy())  # >= 1 MiB each: own pinned outputs
        p = dz.DehazeParams(resize_to=None)
        monkeypatch.setattr(pl, "_PIPE_BATCH_BYTES", 4 * frames[0].nbytes)  # 4 frames per batch: slots get reused
        gc.collect()
        base = pl._pinned_out_bytes
        kept = []
        dz.process_stream(frames, p, sink=kept.append)
        assert pl._pinned_out_bytes == base + 40 * frames[0].nbytes
        snap = [k.copy() for k in kept]
        again = []
        dz.process_stream(iter(frames), p, sink=again.append)   # iterator: immediate copies
        assert all(np.array_equal(a, b) for a, b in zip(kept, snap))
        assert all(np.array_equal(a, b) for a, b in zip(kept, again))
        monkeypatch.setattr(pl, "_PINNED_OUT_BUDGET", 0)        # past the budget: copied out of staging
        plain = []
        dz.process_stream(frames, p, sink=plain.append)
        assert all(np.array_equal(a, b) for a, b in zip(kept, plain))
        assert all(o.flags.owndata for o in plain) and not any(o.flags.owndata for o in kept)
        want = dz.dehaze_frame(frames[17], p)
        assert np.array_equal(kept[17], want)
        view = kept[3][5:9]
        del kept, again
        gc.collect()
        assert pl._pinned_out_bytes == base + frames[0].nbytes   # the view keeps its frame's buffer
        del view
        gc.collect()
        assert pl._pinned_out_bytes == base

    def test_frame_outputs_own_their_memory(self, dz, monkeypatch):
        """dehaze_frame on numpy frames of >= 1 MiB: each result is a view of its own pinned
        tensor (kept results stay intact across later calls, dropped ones return the budget)
        and equals the plain-copy form used past the budget and the CUDA-tensor form."""
        import gc

        import torch

        from paper_2512_16609_b200 import pipeline as pl
        from paper_2512_16609_b200.synthetic import make_frames

        frames = list(make_frames("c3", frames=4, width=800, height=448).numpy())
        p = dz.DehazeParams(resize_to=None)
        gc.collect()
        base = pl._pinned_out_bytes
        kept = [dz.dehaze_frame(f, p) for f in frames]
        assert pl._pinned_out_bytes == base + 4 * frames[0].nbytes
        assert all(o.dtype == np.uint8 and o.shape == frames[0].shape and o.flags.c_contiguous and o.flags.writeable
                   for o in kept)
        snap = [o.copy() for o in kept]
        monkeypatch.setattr(pl, "_PINNED_OUT_BUDGET", 0)
        plain = [dz.dehaze_frame(f, p) for f in frames]
        dev = [dz.dehaze_frame(torch.from_numpy(f).cuda(), p).cpu().numpy() for f in frames]
        assert all(np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, d)
                   for a, b, c, d in zip(kept, snap, plain, dev))
        tel = dz.FrameTelemetry()
        with_tel = dz.dehaze_frame(frames[0], p, tel)
        assert np.array_equal(with_tel, kept[0]) and len(tel.airlights) == 1
        del kept, with_tel
        gc.collect()
        assert pl._pinned_out_bytes == base

    def test_batch_and_host_batch_match_frame_api(self, dz):
        import torch

        from paper_2512_16609_b200.synthetic import make_frames

        frames = make_frames("c3", frames=5, width=160, height=96)
        p = dz.DehazeParams(resize_to=None)
        out_d, air_d = dz.dehaze_batch(frames.cuda(), p)
        out_h, air_h = dz.dehaze_host_batch(frames.pin_memory(), p, chunk=2)
        for i in range(5):
            want = dz.dehaze_frame(frames[i].numpy(), p)
            assert np.array_equal(out_d[i].cpu().numpy(), want)
            assert np.array_equal(out_h[i].numpy(), want)
        assert torch.equal(air_d.cpu(), air_h)

    def test_dehazer_estimator(self, dz):
        frames = np.random.default_rng(5).integers(0, 256, size=(3, 24, 32, 3), dtype=np.uint8)
        est = dz.Dehazer(resize_to=None).fit()
        out = est.transform(frames)
        assert out.shape == frames.shape and out.dtype == np.uint8
        assert np.array_equal(out[1], dz.dehaze_frame(frames[1], dz.DehazeParams(resize_to=None)))
