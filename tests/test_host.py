"""Host-side logic that runs without a GPU: parameter contracts, validation messages,
frame sharding and the airlight-trace exchange (gloo, world_size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.distributed import gather_airlight_trace, shard_range, stabilise_trace
from paper_2512_16609_b200.validation import check_airlight, check_radius, check_u8_frame


class TestParams:
    def test_defaults(self):
        p = DehazeParams()
        assert (p.mode, p.patch_radius, p.top_fraction, p.alpha, p.omega, p.t_min) == \
            ("video", 7, 0.001, 0.8, 0.5, 0.05)
        assert (p.gamma, p.guided_radius, p.guided_eps, p.resize_to, p.white_balance) == \
            (1.2, 40, 1e-3, (640, 480), None)
        q = DehazeParams.for_image()
        assert q.mode == "image" and q.resize_to is None
        assert DehazeParams().balance_enabled() is False and q.balance_enabled() is True

    @pytest.mark.parametrize("field,value", [
        ("mode", "stream"), ("patch_radius", 0), ("patch_radius", 1.5), ("top_fraction", 0.0),
        ("top_fraction", 1.5), ("alpha", 0.0), ("omega", 1.2), ("t_min", 0.0), ("t_min", 1.0),
        ("guided_radius", 0), ("guided_eps", 0.0), ("gamma", 0.0), ("white_balance", "yes"),
        ("resize_to", (0, 480)), ("resize_to", "640x480")])
    def test_validate_rejects(self, field, value):
        with pytest.raises(ValueError):
            DehazeParams(**{field: value}).validate()


class TestValidation:
    def test_u8_frame(self):
        with pytest.raises(ValueError, match="uint8"):
            check_u8_frame(np.zeros((4, 4, 3), np.float32))
        with pytest.raises(ValueError, match=r"H, W, 3"):
            check_u8_frame(np.zeros((4, 4), np.uint8))
        with pytest.raises(ValueError, match="empty"):
            check_u8_frame(np.zeros((0, 4, 3), np.uint8))
        a = np.zeros((4, 6, 3), np.uint8)[:, ::2]
        assert check_u8_frame(a).flags["C_CONTIGUOUS"]

    def test_airlight_and_radius(self):
        with pytest.raises(ValueError, match="airlight"):
            check_airlight((0.0, 0.5, 0.5))
        with pytest.raises(ValueError, match=r"\(3,\)"):
            check_airlight((0.5, 0.5))
        with pytest.raises(ValueError, match="integer"):
            check_radius(1.5)
        with pytest.raises(ValueError, match=">= 0"):
            check_radius(-1)


class TestRouting:
    """Which calls the batched native pipelines cover (pipeline._native_ok) — the rest
    run the per-frame float64 device path; no device is needed to decide."""

    def test_video(self):
        from paper_2512_16609_b200.pipeline import RESIZE_MAX_RADIUS, _native_ok

        assert _native_ok(DehazeParams(resize_to=None), 1080, 1920)
        assert _native_ok(DehazeParams(), 480, 640)                   # resize is a no-op
        assert _native_ok(DehazeParams(), 1080, 1920)                 # default resize path
        assert not _native_ok(DehazeParams(), 1080, 1920, want_maps=True)
        assert _native_ok(DehazeParams(resize_to=None), 1080, 1920, want_maps=True)
        assert _native_ok(DehazeParams(patch_radius=RESIZE_MAX_RADIUS), 100, 100)
        assert not _native_ok(DehazeParams(patch_radius=RESIZE_MAX_RADIUS + 1), 100, 100)
        assert _native_ok(DehazeParams(resize_to=None, patch_radius=60), 100, 100)

    def test_image(self):
        from paper_2512_16609_b200.pipeline import GUIDED_MAX_RADIUS, _native_ok

        img = DehazeParams.for_image()
        assert _native_ok(img, 1080, 1920)
        assert not _native_ok(img, 1080, 1920, want_maps=True)
        assert _native_ok(DehazeParams.for_image(guided_radius=GUIDED_MAX_RADIUS), 64, 64)
        assert not _native_ok(DehazeParams.for_image(guided_radius=GUIDED_MAX_RADIUS + 1), 64, 64)
        assert not _native_ok(DehazeParams.for_image(resize_to=(320, 240)), 1080, 1920)

    def test_working_size(self):
        from paper_2512_16609_b200.engine import FrameEngine

        assert FrameEngine.working_size(DehazeParams(), 1080, 1920) == (480, 640)
        assert FrameEngine.working_size(DehazeParams(resize_to=None), 1080, 1920) == (1080, 1920)
        assert FrameEngine.working_size(DehazeParams(resize_to=(33, 7)), 50, 60) == (7, 33)

    def test_guided_limits_match_the_library(self):
        # the Python routing constants mirror the C++ ones (dhz_internal.h)
        import re

        from paper_2512_16609_b200 import pipeline

        src = open(os.path.join(os.path.dirname(pipeline.__file__), "csrc", "dhz_internal.h")).read()
        assert int(re.search(r"kGuidedMaxRadius = (\d+)", src).group(1)) == pipeline.GUIDED_MAX_RADIUS
        assert int(re.search(r"kResizeMaxRadius = (\d+)", src).group(1)) == pipeline.RESIZE_MAX_RADIUS


class TestSharding:
    @pytest.mark.parametrize("n,world", [(300, 1), (300, 2), (300, 8), (7, 3), (2, 4), (0, 2)])
    def test_shard_range_partitions(self, n, world):
        spans = [shard_range(n, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1

    def test_stabilise_is_the_ema_recurrence(self):
        rng = np.random.default_rng(5)
        tr = torch.from_numpy(rng.uniform(0.5, 0.9, size=(200, 3)))
        for lam in (0.0, 0.3, 0.9):
            got = stabilise_trace(tr, lam).numpy()
            want = np.empty_like(tr.numpy())
            want[0] = tr[0].numpy()
            for f in range(1, 200):
                want[f] = lam * want[f - 1] + (1 - lam) * tr[f].numpy()
            assert np.abs(got - want).max() < 1e-12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(n, rank, world)
        local = torch.arange(lo * 3, hi * 3, dtype=torch.float64).reshape(hi - lo, 3)
        trace = gather_airlight_trace(local, n)
        q.put((rank, trace.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 7])
def test_airlight_trace_allgather_gloo(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(n * 3, dtype=np.float64).reshape(n, 3)
    for r in range(world):
        assert np.array_equal(res[r], want)


def test_stabilise_trace_cpu_matches_oracle(oracle):
    from paper_2512_16609_b200.distributed import stabilise_trace

    rng = np.random.default_rng(5)
    tr = rng.random((97, 3))
    for lam in (0.0, 0.3, 0.95):
        got = stabilise_trace(torch.from_numpy(tr), lam).numpy()
        assert np.array_equal(got, oracle.ema_trace(tr, lam))
    carry = torch.tensor([0.5, 0.6, 0.7], dtype=torch.float64)
    assert np.array_equal(stabilise_trace(torch.from_numpy(tr), 0.7, carry).numpy(),
                          oracle.ema_trace(tr, 0.7, carry.numpy()))
    # causal: smoothing a clip in two pieces with the carry equals smoothing it whole
    whole = stabilise_trace(torch.from_numpy(tr), 0.8)
    head = stabilise_trace(torch.from_numpy(tr[:40]), 0.8)
    tail = stabilise_trace(torch.from_numpy(tr[40:]), 0.8, head[-1])
    assert torch.equal(torch.cat([head, tail]), whole)


def _stab_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_16609_b200.distributed import stabilise_trace

        lo, hi = shard_range(n, rank, world)
        rng = np.random.default_rng(11)
        full = rng.random((n, 3))
        trace = gather_airlight_trace(torch.from_numpy(full[lo:hi].copy()), n)
        q.put((rank, stabilise_trace(trace, 0.9).numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_trace_stabilised_gloo(oracle):
    """world_size 2: every rank ends with the same global smoothed trace, equal to the
    restatement over the unsharded clip (the exchange the GPU ranks make over NCCL)."""
    world, n = 2, 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stab_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.ema_trace(np.random.default_rng(11).random((n, 3)), 0.9)
    for r in range(world):
        assert np.array_equal(res[r], want)
