"""Frame sharding across GPUs and the one cross-GPU exchange (airlight trace all-gather).

The reference runs frames independently (pipeline.py:257-260), so
a clip shards into contiguous frame blocks, one block per rank, with no
data-path collective.  The only exchange is the per-frame airlight trace
(StreamStats.airlight_trace, pipeline.py:252,279,308): each rank all-gathers
its (n_local, 3) float64 block so every rank holds the global trace in frame
order (NCCL over NVLink on GPUs, gloo on CPU for the tests).

``stabilise_trace`` is the optional temporal recurrence named by the
north_star (an EMA over the gathered trace, evaluated as a scan).  It is
NOT part of the reference (SPEC.md:267 lists temporal smoothing as a
non-goal), is off by default and changes outputs when applied.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of frames owned by ``rank`` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(n_frames, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def gather_airlight_trace(local: torch.Tensor, n_frames: int, group=None) -> torch.Tensor:
    """All-gather per-rank (n_local, 3) float64 airlight blocks into the (n_frames, 3) trace.

    Ranks may hold blocks of different sizes (shard_range); blocks are padded
    to the largest one for the collective and trimmed afterwards.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(n_frames, r, world) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros((cap, 3), dtype=torch.float64, device=local.device)
    lo, hi = sizes[rank]
    if local.shape != (hi - lo, 3):
        raise ValueError(f"rank {rank} holds {tuple(local.shape)}, expected ({hi - lo}, 3)")
    buf[: hi - lo] = local
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    parts = [bufs[r][: h - l] for r, (l, h) in enumerate(sizes)]
    return torch.cat(parts, 0)


def stabilise_trace(trace: torch.Tensor, lam: float, carry: torch.Tensor | None = None) -> torch.Tensor:
    """Opt-in EMA recurrence A'_f = lam * A'_{f-1} + (1 - lam) * A_f over an (n, 3) trace.

    CUDA tensors run the library kernel (dhz_ema_airlight); CPU tensors the same
    recurrence in float64 with the same roundings (one per product and sum), so
    both give identical bits.  A'_-1 = ``carry`` when given, else A'_0 = A_0.  Not
    reference behaviour; never applied by default.
    """
    if not 0.0 <= lam < 1.0:
        raise ValueError(f"lam must lie in [0, 1), got {lam}")
    if trace.is_cuda:
        from .engine import ema_airlight

        return ema_airlight(trace, lam, carry=carry)
    a = trace.to(torch.float64).numpy()
    out = a.copy()
    keep, take = float(lam), 1.0 - float(lam)
    prev = None if carry is None else [float(v) for v in carry]
    for f in range(a.shape[0]):
        cur = [float(v) for v in a[f]]
        if prev is not None:
            cur = [keep * p + take * c for p, c in zip(prev, cur)]
        out[f] = cur
        prev = cur
    return torch.from_numpy(out)


def dehaze_sharded(frames_local: torch.Tensor, params, n_frames: int, stabilise: float | None = None,
                   group=None):
    """One rank's part of a frame-sharded clip under torch.distributed (one process per GPU).

    ``frames_local`` is this rank's contiguous block (shard_range) on its GPU.  The
    rank runs the airlight half of the pipeline on its block, all-gathers the
    per-frame airlight (NCCL over NVLink; 24 B/frame, the only exchange), optionally
    smooths the global trace (``stabilise``, not reference behaviour) and recovers
    its block with its slice of the trace.  Returns (out_local, airlight_trace) —
    the trace is global, in frame order, identical on every rank.
    """
    from .engine import engine_for

    if params is None:
        from .pipeline import DehazeParams

        params = DehazeParams()
    params.validate()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n_frames, rank, world)
    if frames_local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {frames_local.shape[0]} frames, shard_range gives {hi - lo}")
    eng = engine_for(frames_local.device)
    raw = eng.phase_airlight(frames_local, params)
    trace = gather_airlight_trace(raw, n_frames, group=group)
    if stabilise is not None:
        trace = stabilise_trace(trace, float(stabilise))
    out = eng.phase_recover(frames_local, params, trace[lo:hi].contiguous())
    return out, trace


class ShardedPipeline:
    """A fixed (frames_local, params) shard replayed step after step under torch.distributed.

    ``dehaze_sharded`` with its two halves captured once as CUDA graphs (the kernels'
    launch gaps go; the buffers are fixed) around an eager NCCL all-gather into a
    preallocated trace — the collective itself is not captured.  ``frames_local`` is
    updated in place between steps.  ``step()`` returns (out_local, airlight_trace);
    both are reused by the next step.
    """

    def __init__(self, frames_local: torch.Tensor, params, n_frames: int, stabilise: float | None = None,
                 group=None):
        from .engine import FrameEngine

        params.validate()
        self.group = group
        self.stabilise = None if stabilise is None else float(stabilise)
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        sizes = [shard_range(n_frames, r, world) for r in range(world)]
        self.lo, self.hi = sizes[rank]
        n = self.hi - self.lo
        if frames_local.shape[0] != n:
            raise ValueError(f"rank {rank} holds {frames_local.shape[0]} frames, shard_range gives {n}")
        dev = frames_local.device
        cap = max(hi - lo for lo, hi in sizes)
        self.frames = frames_local
        self._pad = torch.zeros((cap, 3), dtype=torch.float64, device=dev)   # this rank's block, padded
        self._air_raw = self._pad[:n]
        self._gathered = torch.empty((world * cap, 3), dtype=torch.float64, device=dev)
        self._pick = None
        if any(hi - lo != cap for lo, hi in sizes):  # uneven blocks: drop the padding rows
            self._pick = torch.tensor([r * cap + i for r, (lo, hi) in enumerate(sizes) for i in range(hi - lo)],
                                      dtype=torch.int64, device=dev)
        self._air_in = torch.empty((n, 3), dtype=torch.float64, device=dev)
        h, w = int(frames_local.shape[1]), int(frames_local.shape[2])
        H, W = FrameEngine.working_size(params, h, w)
        self.out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=dev)
        self._eng = FrameEngine(dev)  # private engine: the graphs keep its workspace
        self._g1 = self._g2 = None
        if n:
            first = lambda: self._eng.phase_airlight(self.frames, params, airlight=self._air_raw)  # noqa: E731
            second = lambda: self._eng.phase_recover(self.frames, params, self._air_in, out=self.out)  # noqa: E731
            first()  # eager warm-up: workspace, thresholds, kernel attributes
            self._air_in.copy_(self._air_raw)
            second()
            torch.cuda.synchronize(dev)
            self._g1, self._g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(self._g1):
                first()
            with torch.cuda.graph(self._g2):
                second()
            torch.cuda.synchronize(dev)

    def step(self):
        if self._g1 is not None:
            self._g1.replay()
        dist.all_gather_into_tensor(self._gathered, self._pad, group=self.group)
        trace = self._gathered if self._pick is None else self._gathered.index_select(0, self._pick)
        if self.stabilise is not None:
            trace = stabilise_trace(trace, self.stabilise)
        if self._g2 is not None:
            self._air_in.copy_(trace[self.lo:self.hi])
            self._g2.replay()
        return self.out, trace
