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


def stabilise_trace(trace: torch.Tensor, lam: float) -> torch.Tensor:
    """Opt-in EMA recurrence A'_f = lam * A'_{f-1} + (1 - lam) * A_f, A'_0 = A_0, as a scan.

    Closed form A'_f = lam^f A_0 + (1-lam) sum_{j=1..f} lam^(f-j) A_j, evaluated
    with a cumulative sum of lam^-j-scaled terms in float64 (blocked to keep
    lam^-j in range).  Not reference behaviour; never applied by default.
    """
    if not 0.0 <= lam < 1.0:
        raise ValueError(f"lam must lie in [0, 1), got {lam}")
    n = trace.shape[0]
    if n == 0 or lam == 0.0:
        return trace.clone()
    out = torch.empty_like(trace)
    block = 64
    carry = trace[0].clone()
    out[0] = carry
    f = 1
    while f < n:
        m = min(block, n - f)
        j = torch.arange(1, m + 1, dtype=trace.dtype, device=trace.device)
        w = lam ** (-j)                                   # lam^-j, j = 1..m
        terms = (1.0 - lam) * trace[f: f + m] * w[:, None]
        pref = torch.cumsum(terms, 0) * (lam ** j)[:, None]
        out[f: f + m] = pref + (lam ** j)[:, None] * carry
        carry = out[f + m - 1].clone()
        f += m
    return out
