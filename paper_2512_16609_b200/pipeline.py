"""Per-frame dehazing pipeline and stream orchestration (drop-in for reference pipeline.py).

Same public surface as ``/root/reference/pkg/src/dehaze/pipeline.py``:
``DehazeParams`` (:52-114), ``FrameTelemetry`` (:117-150), ``StreamStats``
(:153-160), ``dehaze_frame`` (:163-216), ``dehaze_image`` (:219-229),
``process_stream`` (:232-308), ``VIDEO_STAGES`` / ``IMAGE_STAGES`` (:39-49).

The compute runs on the GPU through libdehaze_b200.so:

* u8 frames at native size (``resize_to`` None or equal to the frame size):
  the fused batch pipeline (engine.FrameEngine, one C-ABI call per batch);
* frames that need the bilinear resize (the reference default
  ``resize_to=(640, 480)``) go through the float64 device path
  (``floatpath``), which keeps the reference's float64 semantics.

``process_stream`` batches frames on the device instead of fanning them out to
CPU threads; ``workers`` keeps its contract (validated, results bit-identical
for every value) but no longer changes the schedule.  Additions (all default
to reference behaviour): ``dehaze_batch`` for device-resident batches, and the
``device=`` keyword.
"""

from __future__ import annotations

import time
from contextlib import contextmanager
from dataclasses import dataclass, field, replace

import numpy as np

from .estimation import (
    DEFAULT_ALPHA,
    DEFAULT_GUIDED_EPS,
    DEFAULT_GUIDED_RADIUS,
    DEFAULT_OMEGA,
    DEFAULT_PATCH_RADIUS,
    DEFAULT_T_MIN,
    DEFAULT_TOP_FRACTION,
)
from .recover import DEFAULT_GAMMA
from .validation import check_u8_frame

DEFAULT_STREAM_SIZE = (640, 480)

VIDEO_STAGES = (
    "resize",
    "channel_min",
    "min_filter",
    "airlight",
    "transmission",
    "recover",
    "postprocess",
    "output",
)
IMAGE_STAGES = VIDEO_STAGES[:5] + ("guided_filter",) + VIDEO_STAGES[5:]

# How fused device work is attributed to the reference's stage names: the time
# between consecutive ABI events goes to the first stage of each group; the
# other stages of the group are recorded with 0.0 s (they run inside the same
# kernel).  Event order: see include/dehaze_b200.h (DHZ_N_EVENTS).
_STAGE_GROUPS_VIDEO = (("min_filter", "resize", "channel_min"), ("airlight",), ("transmission",),
                       ("recover", "postprocess", "output"))
_STAGE_GROUPS_IMAGE = (("min_filter", "resize", "channel_min"), ("airlight",),
                       ("guided_filter", "transmission"), ("recover", "postprocess", "output"))


@dataclass(frozen=True)
class DehazeParams:
    """Hyperparameters for the dehazing pipeline (reference pipeline.py:52-114).

    mode selects the stage set: "video" (no transmission refinement, frames
    resized to resize_to) or "image" (guided-filter refinement, native
    resolution unless resize_to is set). white_balance=None means the mode
    default: off for video, on for image.
    """

    mode: str = "video"
    patch_radius: int = DEFAULT_PATCH_RADIUS
    top_fraction: float = DEFAULT_TOP_FRACTION
    alpha: float = DEFAULT_ALPHA
    omega: float = DEFAULT_OMEGA
    t_min: float = DEFAULT_T_MIN
    guided_radius: int = DEFAULT_GUIDED_RADIUS
    guided_eps: float = DEFAULT_GUIDED_EPS
    gamma: float = DEFAULT_GAMMA
    white_balance: bool = None
    resize_to: tuple = DEFAULT_STREAM_SIZE

    @classmethod
    def for_image(cls, **overrides):
        """Parameters for single-image work: refine t, keep native size."""
        overrides.setdefault("mode", "image")
        overrides.setdefault("resize_to", None)
        return cls(**overrides)

    def validate(self):
        if self.mode not in ("video", "image"):
            raise ValueError(f"mode must be 'video' or 'image', got {self.mode!r}")
        if int(self.patch_radius) != self.patch_radius or self.patch_radius < 1:
            raise ValueError(f"patch_radius must be an integer >= 1, got {self.patch_radius}")
        if not 0.0 < self.top_fraction <= 1.0:
            raise ValueError(f"top_fraction must lie in (0, 1], got {self.top_fraction}")
        if not 0.0 < self.alpha <= 1.0:
            raise ValueError(f"alpha must lie in (0, 1], got {self.alpha}")
        if not 0.0 < self.omega <= 1.0:
            raise ValueError(f"omega must lie in (0, 1], got {self.omega}")
        if not 0.0 < self.t_min < 1.0:
            raise ValueError(f"t_min must lie in (0, 1), got {self.t_min}")
        if int(self.guided_radius) != self.guided_radius or self.guided_radius < 1:
            raise ValueError(f"guided_radius must be an integer >= 1, got {self.guided_radius}")
        if not self.guided_eps > 0.0:
            raise ValueError(f"guided_eps must be positive, got {self.guided_eps}")
        if not self.gamma > 0.0:
            raise ValueError(f"gamma must be positive, got {self.gamma}")
        if self.white_balance not in (None, True, False):
            raise ValueError(f"white_balance must be None or bool, got {self.white_balance!r}")
        if self.resize_to is not None:
            try:
                w, h = self.resize_to
            except (TypeError, ValueError):
                raise ValueError(f"resize_to must be None or (width, height), got {self.resize_to!r}")
            if int(w) != w or int(h) != h or w < 1 or h < 1:
                raise ValueError(f"resize_to must hold positive integers, got {self.resize_to!r}")
        return self

    def balance_enabled(self):
        if self.white_balance is None:
            return self.mode == "image"
        return self.white_balance


class FrameTelemetry:
    """Per-stage time and call counts, plus the airlight trace (reference pipeline.py:117-150).

    Stage times of the fused device path are CUDA-event times (seconds); see
    ``_STAGE_GROUPS_*`` for how fused kernels map onto the stage names.
    """

    def __init__(self, capture_maps=False):
        self.timings = {}
        self.counts = {}
        self.airlights = []
        self.capture_maps = capture_maps
        self.maps = {}

    @contextmanager
    def stage(self, name):
        start = time.perf_counter()
        try:
            yield
        finally:
            self.add_time(name, time.perf_counter() - start)

    def add_time(self, name, seconds):
        self.timings.setdefault(name, []).append(float(seconds))
        self.counts[name] = self.counts.get(name, 0) + 1

    def record_airlight(self, airlight):
        self.airlights.append(np.asarray(airlight, dtype=np.float64).copy())

    def record_map(self, name, m):
        if self.capture_maps:
            self.maps[name] = np.array(m, dtype=np.float64, copy=True)

    def total_time(self, name):
        return sum(self.timings.get(name, ()))


@dataclass
class StreamStats:
    """Summary of one stream run."""

    frame_count: int
    wall_time: float
    fps: float
    airlight_trace: list = field(default_factory=list)


def _needs_resize(params, h, w):
    if params.resize_to is None:
        return False
    rw, rh = params.resize_to
    return (int(rw), int(rh)) != (w, h)


GUIDED_MAX_RADIUS = 255  # dhz::kGuidedMaxRadius (fused guided filter: 2r < 512 columns per strip)


RESIZE_MAX_RADIUS = 32  # dhz::kResizeMaxRadius (tile halo of the resize path's erosion)


def _native_ok(params, h, w, want_maps=False):
    """Whether the batched native pipeline (dhz_frames_u8 / dhz_frames_resize_u8)
    covers this call: video mode at native size or resized (patch radius up to
    RESIZE_MAX_RADIUS), image mode at native size (guided radius up to
    GUIDED_MAX_RADIUS).  Map capture outside plain native-size video, image mode
    with a resize, and larger radii use the per-frame float64 device path."""
    if _needs_resize(params, h, w):
        return params.mode == "video" and int(params.patch_radius) <= RESIZE_MAX_RADIUS and not want_maps
    if params.mode == "image":
        return int(params.guided_radius) <= GUIDED_MAX_RADIUS and not want_maps
    return True


def _as_device_batch(frames_np, device):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(frames_np))
    return t.to(device=device, non_blocking=False)


def _check_stabilise(stabilise):
    """stabilise=None (reference behaviour) or the EMA weight lam in [0, 1)."""
    if stabilise is None:
        return None
    lam = float(stabilise)
    if not 0.0 <= lam < 1.0:
        raise ValueError(f"stabilise must be None or lie in [0, 1), got {stabilise!r}")
    return lam


def _device_list(devices):
    """devices=None -> None; else a list of torch CUDA devices (repeats allowed)."""
    if devices is None:
        return None
    import torch

    out = []
    for d in devices:
        d = torch.device("cuda", d) if isinstance(d, int) else torch.device(d)
        if d.type != "cuda":
            raise ValueError(f"devices must be CUDA devices, got {d}")
        out.append(torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device()))
    if not out:
        raise ValueError("devices must name at least one CUDA device")
    return out


_groups: dict = {}


def _group(devs):
    from .engine import DeviceGroup

    import threading

    key = (tuple(d.index for d in devs), threading.get_ident())
    g = _groups.get(key)
    if g is None:
        g = _groups[key] = DeviceGroup(devs)
    return g


def _run_native(batch, params, telemetry=None, keep_maps=False):
    """batch: (n, H, W, 3) uint8 CUDA tensor at its working size."""
    import torch

    from .engine import engine_for

    eng = engine_for(batch.device)
    if telemetry is None:
        return eng.run(batch, params, keep_maps=keep_maps)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    res = eng.run(batch, params, keep_maps=keep_maps, events=evs)
    evs[-1].synchronize()
    groups = _STAGE_GROUPS_IMAGE if params.mode == "image" else _STAGE_GROUPS_VIDEO
    for i, grp in enumerate(groups):
        dt = evs[i].elapsed_time(evs[i + 1]) / 1000.0
        telemetry.add_time(grp[0], max(dt, 0.0))
        for other in grp[1:]:
            telemetry.add_time(other, 0.0)
    return res


def _frame_roundtrip(frame, params, telemetry, dev):
    """One numpy frame through the native pipeline: (output array, airlight array).  The
    frame is staged in pinned memory (H2D asynchronous), the output lands in its own
    pinned host tensor and is returned as a numpy view of it (budgeted like
    process_stream's outputs; a plain copy past the budget)."""
    import torch

    from .engine import FrameEngine

    h, w = int(frame.shape[0]), int(frame.shape[1])
    OH, OW = FrameEngine.working_size(params, h, w)
    with torch.cuda.device(dev):
        hin = torch.empty((1, h, w, 3), dtype=torch.uint8, pin_memory=True)
        _par_copy(hin[0], torch.from_numpy(frame))
        din = hin.to(dev, non_blocking=True)
        out, air = _run_native(din, params, telemetry)[:2]
        nbytes = OH * OW * 3
        if nbytes >= _PINNED_OUT_MIN and _pinned_out_take(nbytes):
            import weakref

            hout = torch.empty((OH, OW, 3), dtype=torch.uint8, pin_memory=True)
            hair = torch.empty(3, dtype=torch.float64, pin_memory=True)
            hout.copy_(out[0], non_blocking=True)
            hair.copy_(air[0], non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            arr = hout.numpy()
            weakref.finalize(arr, _pinned_out_release, nbytes)
            return arr, hair.numpy().copy()
        return out[0].cpu().numpy(), air[0].cpu().numpy()


def _device():
    import torch

    from . import _native

    _native.lib()  # fail loudly without the library / a CUDA device
    return torch.device("cuda", torch.cuda.current_device())


def dehaze_frame(frame, params=None, telemetry=None):
    """Dehaze one interleaved uint8 RGB frame; returns a uint8 frame (reference pipeline.py:163-216).

    Accepts a numpy array (returns numpy) or a CUDA uint8 tensor (returns a
    CUDA tensor, no host copies).  Pure: equal inputs give bit-equal outputs.
    """
    if params is None:
        params = DehazeParams()
    params.validate()
    tel = telemetry if telemetry is not None else FrameTelemetry()
    frame = check_u8_frame(frame)
    is_tensor = not isinstance(frame, np.ndarray)
    dev = frame.device if is_tensor else _device()
    h, w = int(frame.shape[0]), int(frame.shape[1])
    if not _native_ok(params, h, w, tel.capture_maps):
        from .floatpath import dehaze_float_frame

        out, airlight, maps = dehaze_float_frame(frame if is_tensor else _as_device_batch(frame, dev),
                                                 params, tel)
    elif not is_tensor and not tel.capture_maps:
        # numpy in, numpy out: pinned staging in, the output in its own pinned tensor (see
        # _StreamPipe), one synchronisation; stage events only when the caller asked for them
        out_np, a_host = _frame_roundtrip(frame, params, telemetry, dev)
        tel.record_airlight(a_host)
        return out_np
    else:
        batch = frame[None] if is_tensor else _as_device_batch(frame[None], dev)
        want_maps = tel.capture_maps
        res = _run_native(batch, params, tel, keep_maps=want_maps)
        out, airlight = res[0][0], res[1][0]
        maps = None
        if want_maps:
            from .floatpath import maps_from_native

            maps = maps_from_native(batch[0], res[2], airlight, params)
    a_host = airlight.detach().cpu().numpy()
    tel.record_airlight(a_host)
    if maps is not None:
        for name in ("dark", "transmission_coarse", "transmission"):
            tel.record_map(name, maps[name])
    if is_tensor:
        return out
    return out.cpu().numpy()


def dehaze_image(frame, params=None, telemetry=None):
    """Dehaze a single image at native resolution with refinement on (reference pipeline.py:219-229)."""
    if params is None:
        params = DehazeParams.for_image()
    elif params.mode != "image":
        params = replace(params, mode="image")
    return dehaze_frame(frame, params, telemetry)


def dehaze_batch(frames, params=None, out=None, devices=None, stabilise=None):
    """Dehaze a device-resident batch (n, H, W, 3) uint8 CUDA tensor in one pipeline launch.

    Returns (out, airlight) CUDA tensors: out (n, H', W', 3) uint8, airlight
    (n, 3) float64, with (H', W') the working size (resize_to in video mode).
    Calls the batched native path does not cover (see _native_ok) run the
    per-frame float64 device path.

    ``devices`` (list of CUDA devices, repeats allowed): shard the batch by frame
    over them (contiguous blocks; the airlight trace is all-gathered through
    dhz_allgather_airlight); results are bit-identical to one device.
    ``stabilise=lam`` (opt-in, NOT reference behaviour, reference SPEC.md:267):
    smooth the airlight trace with A'_f = lam A'_{f-1} + (1 - lam) A_f before the
    recovery; the returned airlight is A'.
    """
    if params is None:
        params = DehazeParams()
    params.validate()
    lam = _check_stabilise(stabilise)
    devs = _device_list(devices)
    n, h, w = int(frames.shape[0]), int(frames.shape[1]), int(frames.shape[2])
    if (devs is not None or lam is not None) and not _native_ok(params, h, w):
        raise ValueError("devices= / stabilise= need a call the batched native pipeline covers "
                         "(see _native_ok: image mode with a resize, map capture, guided_radius > "
                         f"{GUIDED_MAX_RADIUS} or patch_radius > {RESIZE_MAX_RADIUS} after a resize are not)")
    if devs is not None:
        return _group(devs).run(frames, params, out=out, stabilise=lam)
    if not _native_ok(params, h, w):
        import torch

        from .floatpath import dehaze_float_frame

        outs, airs = [], []
        for i in range(n):
            o, a, _ = dehaze_float_frame(frames[i], params, None)
            outs.append(o)
            airs.append(a)
        if n == 0:
            oh, ow = (h, w) if params.resize_to is None else (int(params.resize_to[1]), int(params.resize_to[0]))
            return (torch.empty((0, oh, ow, 3), dtype=torch.uint8, device=frames.device),
                    torch.empty((0, 3), dtype=torch.float64, device=frames.device))
        return torch.stack(outs), torch.stack(airs)
    from .engine import engine_for

    return engine_for(frames.device).run(frames, params, out=out, stabilise=lam)


class _HostPipe:
    """Per-(device, shape) ring of stream slots for host-resident batches."""

    def __init__(self, dev, chunk, H, W, OH, OW, slots=3):
        import torch

        from .engine import FrameEngine

        self.streams = [torch.cuda.Stream(dev) for _ in range(slots)]
        self.engines = [FrameEngine(dev) for _ in range(slots)]
        self.din = [torch.empty((chunk, H, W, 3), dtype=torch.uint8, device=dev) for _ in range(slots)]
        self.dout = [torch.empty((chunk, OH, OW, 3), dtype=torch.uint8, device=dev) for _ in range(slots)]
        self.dair = [torch.empty((chunk, 3), dtype=torch.float64, device=dev) for _ in range(slots)]
        self.carry = torch.zeros(3, dtype=torch.float64, device=dev)  # stabilise: A' carried across chunks


_host_pipes: dict = {}


def dehaze_host_batch(frames, params=None, out=None, airlight=None, chunk=None, devices=None, stabilise=None):
    """Dehaze a HOST batch (n, H, W, 3) uint8 torch tensor (pinned for overlap) end to end.

    Frames move to the GPU in chunks on a ring of streams: H2D copy, fused
    pipeline and D2H copy of chunk c overlap those of chunks c-1 and c+1.
    Returns (out, airlight) host tensors (pinned when allocated here); out has
    the working size (resize_to in video mode).  ``devices``: one ring per device
    over its contiguous block of frames (all devices copy and compute at once);
    ``stabilise``: as in dehaze_batch (the recurrence runs chunk by chunk in frame
    order, carrying A' across chunks).
    """
    import torch

    if params is None:
        params = DehazeParams()
    params.validate()
    lam = _check_stabilise(stabilise)
    devs = _device_list(devices)
    n, H, W = int(frames.shape[0]), int(frames.shape[1]), int(frames.shape[2])
    if (devs is not None or lam is not None) and not _native_ok(params, H, W):
        raise ValueError("devices= / stabilise= need a call the batched native pipeline covers (see _native_ok)")
    if devs is not None and lam is not None and len(devs) > 1:
        # the recurrence needs every earlier frame's airlight: keep the shards resident
        o, a = _group(devs).run(frames, params, stabilise=lam)
        o, a = o.cpu(), a.cpu()
        if out is not None:
            out.copy_(o)
            o = out
        if airlight is not None:
            airlight.copy_(a)
            a = airlight
        return o, a
    if not _native_ok(params, H, W):
        # resize / very wide guided windows: float64 device path, frame by frame
        o, a = dehaze_batch(frames.to(_device()), params)
        if out is not None:
            out.copy_(o)
            o = out
        if airlight is not None:
            airlight.copy_(a)
            a = airlight
        return o.cpu() if o.is_cuda else o, a.cpu() if a.is_cuda else a
    from .distributed import shard_range
    from .engine import FrameEngine

    devs = devs if devs is not None else [_device()]
    OH, OW = FrameEngine.working_size(params, H, W)
    if out is None:
        out = torch.empty((n, OH, OW, 3), dtype=torch.uint8, pin_memory=True)
    if airlight is None:
        airlight = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
    if n == 0:
        return out, airlight
    if chunk is None:
        # ~96 MiB of input per ring step (tools/host_chunk_probe.py: C4 2-4 frames 63 ms vs
        # 66.7 ms one frame per step; C3 16 frames 39.9 vs 40.4 ms for 7)
        chunk = max(1, min(n, (96 << 20) // (3 * H * W)))
    import threading

    # per (device, thread), like engine_for: concurrent callers never share staging buffers;
    # a device listed twice gets two rings
    pipes, plans = [], []
    for i, dev in enumerate(devs):
        key = (dev.index, i, threading.get_ident(), chunk, H, W, OH, OW)
        pipe = _host_pipes.get(key)
        if pipe is None:
            pipe = _host_pipes[key] = _HostPipe(dev, chunk, H, W, OH, OW)
        cur = torch.cuda.current_stream(dev)
        for st in pipe.streams:
            st.wait_stream(cur)
        lo, hi = shard_range(n, i, len(devs))
        pipes.append(pipe)
        plans.append(list(range(lo, hi, chunk)))
    carry = None  # stabilise: A' of the last frame before the chunk (single device: in frame order)
    carry_ev = None
    for c in range(max(len(p) for p in plans)):
        for i, pipe in enumerate(pipes):  # interleave: every device's ring advances each round
            if c >= len(plans[i]):
                continue
            lo = plans[i][c]
            hi = min(lo + chunk, shard_range(n, i, len(devs))[1])
            s = c % len(pipe.streams)
            st = pipe.streams[s]
            m = hi - lo
            with torch.cuda.stream(st):
                pipe.din[s][:m].copy_(frames[lo: hi], non_blocking=True)
                if lam is not None and carry_ev is not None:
                    st.wait_event(carry_ev)
                pipe.engines[s].run(pipe.din[s][:m], params, out=pipe.dout[s][:m], airlight=pipe.dair[s][:m],
                                    stream=st, stabilise=lam, carry=carry)
                if lam is not None:
                    carry = pipe.carry
                    carry.copy_(pipe.dair[s][m - 1], non_blocking=True)
                    carry_ev = torch.cuda.Event()
                    carry_ev.record(st)
                out[lo: hi].copy_(pipe.dout[s][:m], non_blocking=True)
                airlight[lo: hi].copy_(pipe.dair[s][:m], non_blocking=True)
    for pipe in pipes:
        for st in pipe.streams:
            st.synchronize()
    return out, airlight


_STREAM_BATCH_BYTES = 256 << 20   # float path: ~256 MiB of input frames per device launch
_COPY_THREADS = max(1, min(8, (__import__("os").cpu_count() or 1)))
_copy_pool = None


def _pool():
    """Host-copy threads of process_stream (numpy/torch copies release the GIL)."""
    global _copy_pool
    if _copy_pool is None:
        from concurrent.futures import ThreadPoolExecutor

        _copy_pool = ThreadPoolExecutor(max_workers=_COPY_THREADS, thread_name_prefix="dhz-copy")
    return _copy_pool


def _par_copy(dst, src):
    """dst.copy_(src) for host tensors, split over the copy threads when large; returns
    when the copy is complete."""
    nb = src.numel() * src.element_size()
    # measured on the B200 box's host (tools/stream_copy_probe.py): splitting a 6 MB 1080p
    # frame over threads loses to one memcpy (dispatch cost); 4K/8K frames gain
    k = min(_COPY_THREADS, nb >> 22) if nb >= (8 << 20) else 1  # >= 4 MiB per piece
    if k < 2:
        dst.copy_(src)
        return
    d, s_ = dst.reshape(-1), src.reshape(-1)
    n = d.numel()
    cuts = [n * i // k for i in range(k + 1)]
    list(_pool().map(lambda i: d[cuts[i]:cuts[i + 1]].copy_(s_[cuts[i]:cuts[i + 1]]), range(k)))
_STREAM_BATCH_MAX = 256
_PIPE_BATCH_BYTES = 48 << 20      # native path: input bytes per pipelined batch
_PIPE_SLOTS = 4                  # one slot's copies pending, three batches in flight (tools/ps_sweep.py)
# Fresh output frames are handed out as numpy views of their own pinned host tensors (the
# D2H copy lands in them directly: no staging copy, no first-touch page faults) while the
# bytes still held by the caller stay under this budget; past it (a sink that keeps every
# frame of a long clip) outputs are copied out of the slot's staging into plain arrays.
_PINNED_OUT_BUDGET = int(__import__("os").environ.get("DHZ_PINNED_OUT_BYTES", 1 << 30))
_PINNED_OUT_MIN = 1 << 20   # smaller frames (VGA): the staging copy is cheaper than a pinned tensor each
_pinned_out_lock = __import__("threading").Lock()
_pinned_out_bytes = 0


def _pinned_out_take(nbytes):
    global _pinned_out_bytes
    with _pinned_out_lock:
        if _pinned_out_bytes + nbytes > _PINNED_OUT_BUDGET:
            return False
        _pinned_out_bytes += nbytes
        return True


def _pinned_out_release(nbytes):
    global _pinned_out_bytes
    with _pinned_out_lock:
        _pinned_out_bytes -= nbytes


_pipe_cache = __import__("threading").local()   # .entry = (key, pipe): the calling thread's last pipe


def _acquire_pipe(devs, params, shape, stabilise, n_hint):
    """process_stream's pipe: the thread's previous one when the geometry is the same
    (staging, device buffers, streams and engines are reused: a one-frame stream costs no
    set-up), a new one otherwise or when that one is busy (a sink calling process_stream)."""
    probe_batch = max(1, min(_STREAM_BATCH_MAX, _PIPE_BATCH_BYTES // (3 * shape[0] * shape[1])))
    if n_hint is not None:
        probe_batch = max(1, min(probe_batch, -(-int(n_hint) // _PIPE_SLOTS)))
    from .engine import FrameEngine

    key = (tuple((d.type, d.index) for d in devs), tuple(shape), FrameEngine.working_size(params, shape[0], shape[1]),
           probe_batch)
    entry = getattr(_pipe_cache, "entry", None)
    if entry is not None and entry[0] == key and not entry[1].busy:
        pipe = entry[1]
        pipe.reset(params, stabilise)
    else:
        pipe = _StreamPipe(devs, params, shape, stabilise=stabilise, n_hint=n_hint)
        if entry is None or not entry[1].busy:
            _pipe_cache.entry = (key, pipe)
    pipe.busy = True
    return pipe


class _StreamPipe:
    """process_stream's pipelined batches on the native path.

    Each slot owns pinned host staging (input, output, airlight), device buffers,
    a stream and an engine.  Frames are copied into a slot's pinned input as they
    arrive; a full slot is submitted (H2D, fused pipeline, D2H, all async on its
    stream) and the host goes on filling the next slot, so PCIe transfers and
    kernels of batch k overlap the host copies of batch k+1.  Slots are drained
    (outputs handed to the sink) in submission order, which keeps frame order.
    With several devices the slots alternate between them (slot k on device
    k mod ndev), so consecutive batches run on different GPUs at the same time.
    With ``stabilise`` each batch's recurrence starts from the previous batch's
    last A' (an event chain across the slots; the carry hops devices if needed).
    """

    def __init__(self, devs, params, shape, fresh=True, stabilise=None, n_hint=None):
        import torch

        from .engine import FrameEngine

        H, W, _ = shape
        OH, OW = FrameEngine.working_size(params, H, W)
        self.batch = max(1, min(_STREAM_BATCH_MAX, _PIPE_BATCH_BYTES // (3 * H * W)))
        if n_hint is not None:  # a short clip of known length: slots no larger than its share
            self.batch = max(1, min(self.batch, -(-int(n_hint) // _PIPE_SLOTS)))
        self.params = params
        self.lam = stabilise
        self.out_shape = (OH, OW, 3)
        S, B = _PIPE_SLOTS * len(devs), self.batch
        sdev = [devs[k % len(devs)] for k in range(S)]
        pin = dict(dtype=torch.uint8, pin_memory=True)
        self.hin = [torch.empty((B, H, W, 3), **pin) for _ in range(S)]
        self.hout = [None] * S   # output staging, allocated on first use (outputs normally own their memory)
        self._hout_shape = (B, OH, OW, 3)
        self.hair = [torch.empty((B, 3), dtype=torch.float64, pin_memory=True) for _ in range(S)]
        self.din = [torch.empty((B, H, W, 3), dtype=torch.uint8, device=d) for d in sdev]
        self.dout = [torch.empty((B, OH, OW, 3), dtype=torch.uint8, device=d) for d in sdev]
        self.dair = [torch.empty((B, 3), dtype=torch.float64, device=d) for d in sdev]
        self.carry = [torch.zeros(3, dtype=torch.float64, device=d) for d in sdev]
        self.streams = [torch.cuda.Stream(d) for d in sdev]
        self.engines = [FrameEngine(d) for d in sdev]
        self.events = [torch.cuda.Event() for _ in range(S)]
        self.inflight = [0] * S
        self.slot = 0
        self.fill = 0
        self.prev = None  # (slot, rows) of the last submitted batch (stabilise carry source)
        self.fresh = fresh  # False: emit views of the pinned output (the consumer copies at once)
        self._emit = None
        self._pending = None       # (slot, rows, copy futures) of a closed batch not launched yet
        self.busy = False          # held by a running process_stream (see _acquire_pipe)
        self.own = [None] * S      # per slot: the batch's own pinned output tensors (fresh mode)
        self.lazy = [[] for _ in range(S)]  # per slot: (row, frame) copies deferred to submit()
        self.out_bytes = OH * OW * 3

    def reset(self, params, stabilise):
        """Ready a cached pipe for another stream: wait for anything an aborted stream left
        in flight, return its share of the pinned-output budget, clear the ring."""
        for f in (self._pending[2] if self._pending is not None else ()):
            try:
                f.result()
            except Exception:
                pass
        for s, m in enumerate(self.inflight):
            if m:
                self.events[s].synchronize()
            if self.own[s] is not None:
                _pinned_out_release(len(self.own[s]) * self.out_bytes)
                self.own[s] = None
            self.inflight[s] = 0
            self.lazy[s].clear()
        self.params, self.lam = params, stabilise
        self.slot = self.fill = 0
        self.prev = self._pending = self._emit = None

    def next_input(self, emit=None):
        """The pinned input frame the next frame goes into (drains the slot's previous batch first)."""
        s = self.slot
        if self.fill == 0 and self.inflight[s]:
            self.drain(s, emit if emit is not None else self._emit)
        return self.hin[s][self.fill]

    def commit(self, emit):
        self._emit = emit
        self.fill += 1
        if self.fill == self.batch:
            self.submit()

    def put(self, frame, emit, persistent=False):
        """Stage one frame.  ``persistent``: the caller keeps ``frame`` alive and unchanged
        until the stream ends (a list of frames), so its copy into the pinned slot may wait
        for submit(), where the batch's copies run side by side on the copy threads;
        otherwise the copy is done before returning (the source may reuse its buffer)."""
        import torch

        dst = self.next_input(emit)
        if persistent and frame.nbytes >= (1 << 19):
            self.lazy[self.slot].append((dst, frame))
        else:
            _par_copy(dst, torch.from_numpy(frame))
        self.commit(emit)

    def submit(self):
        """Close the slot being filled.  Its deferred staging copies start on the copy
        threads and the ring moves on at once; the batch is launched (H2D, pipeline, D2H)
        at the next submit()/finish(), after the previously closed batch's copies — so
        the host copies of batch k+1 run while batch k is being enqueued."""
        import torch

        s, m = self.slot, self.fill
        if m == 0:
            self._launch_pending()
            return
        lazy, futs = self.lazy[s], None
        if lazy:
            if len(lazy) > 1:
                futs = [_pool().submit(job[0].copy_, torch.from_numpy(job[1])) for job in lazy]
            else:
                _par_copy(lazy[0][0], torch.from_numpy(lazy[0][1]))
            lazy.clear()
        self.slot = (s + 1) % len(self.hin)
        self.fill = 0
        self._launch_pending()
        if futs is None:
            self._launch(s, m)
        else:
            self._pending = (s, m, futs)

    def _launch_pending(self):
        if self._pending is not None:
            s, m, futs = self._pending
            self._pending = None
            for f in futs:
                f.result()
            self._launch(s, m)

    def _launch(self, s, m):
        import torch

        own = None
        if self.fresh and self.out_bytes >= _PINNED_OUT_MIN and _pinned_out_take(m * self.out_bytes):
            own = [torch.empty(self.out_shape, dtype=torch.uint8, pin_memory=True) for _ in range(m)]
        self.own[s] = own
        st = self.streams[s]
        with torch.cuda.stream(st):
            self.din[s][:m].copy_(self.hin[s][:m], non_blocking=True)
            carry = None
            if self.lam is not None and self.prev is not None:
                p, pm = self.prev
                st.wait_event(self.events[p])
                self.carry[s].copy_(self.dair[p][pm - 1], non_blocking=True)
                carry = self.carry[s]
            self.engines[s].run(self.din[s][:m], self.params, out=self.dout[s][:m], airlight=self.dair[s][:m],
                                stream=st, stabilise=self.lam, carry=carry)
            if own is not None:
                for i in range(m):
                    own[i].copy_(self.dout[s][i], non_blocking=True)
            else:
                if self.hout[s] is None:
                    self.hout[s] = torch.empty(self._hout_shape, dtype=torch.uint8, pin_memory=True)
                self.hout[s][:m].copy_(self.dout[s][:m], non_blocking=True)
            self.hair[s][:m].copy_(self.dair[s][:m], non_blocking=True)
            self.events[s].record(st)
        self.inflight[s] = m
        self.prev = (s, m)

    def drain(self, s, emit):
        import torch

        m = self.inflight[s]
        if not m:
            return
        self.events[s].synchronize()
        own, self.own[s] = self.own[s], None
        if own is not None:  # each frame owns its pinned tensor; the budget follows the arrays' lifetime
            import weakref

            outs = [t.numpy() for t in own]
            for o in outs:
                weakref.finalize(o, _pinned_out_release, self.out_bytes)
            del own
        elif self.fresh:  # the sink may keep them: fresh arrays, filled by the copy threads
            outs = [np.empty(self.out_shape, dtype=np.uint8) for _ in range(m)]
            hout = self.hout[s]
            if m > 1 and outs[0].nbytes >= (1 << 19):
                list(_pool().map(lambda i: torch.from_numpy(outs[i]).copy_(hout[i]), range(m)))
            else:
                for i in range(m):
                    torch.from_numpy(outs[i]).copy_(hout[i])
        else:
            outs = [self.hout[s][i].numpy() for i in range(m)]
        for i in range(m):
            emit(outs[i], self.hair[s][i].numpy().copy())
        self.inflight[s] = 0

    def __del__(self):  # a stream abandoned mid-way (the sink raised): return its share of the budget
        try:
            for s, own in enumerate(self.own):
                if own is not None:
                    _pinned_out_release(len(own) * self.out_bytes)
                    self.own[s] = None
        except Exception:
            pass

    def finish(self, emit):
        self.submit()
        self._launch_pending()
        S = len(self.hin)
        for k in range(S):  # oldest first: the slot after the last submitted one
            self.drain((self.slot + k) % S, emit)


def process_stream(frames, params=None, sink=None, workers=1, devices=None, stabilise=None):
    """Run the pipeline over an iterable of uint8 frames, in order (reference pipeline.py:232-308).

    Frames are validated as they arrive and dehazed in device batches; each
    output frame reaches ``sink`` in input order.  A mid-stream size change
    raises after every frame before it has been dehazed and handed to the sink.
    On the native paths the batches are pipelined (``_StreamPipe``); ``workers``
    keeps the reference's contract (>= 1; results never depend on it).
    Additions (defaults = reference behaviour): ``devices`` spreads consecutive
    batches over several GPUs (the multi-GPU stand-in for the reference's thread
    fan-out, pipeline.py:282-304); ``stabilise=lam`` smooths the airlight trace
    (A'_f = lam A'_{f-1} + (1 - lam) A_f; not reference behaviour),
    and the trace then records A'.
    """
    if params is None:
        params = DehazeParams()
    params.validate()
    workers = int(workers)
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    lam = _check_stabilise(stabilise)
    devs = _device_list(devices)

    try:  # a sequence of known length sizes the pipelined batches of a short clip
        n_hint = len(frames)
    except TypeError:
        n_hint = None
    # a list's frames stay alive and unchanged for the whole call: their staging copies may be
    # deferred and run in parallel (an iterator may reuse its buffer, so it is copied at once)
    persistent = isinstance(frames, (list, tuple)) and __import__("os").environ.get("DHZ_PS_LAZY", "1") != "0"
    trace = []
    count = 0
    expected_shape = None
    start = time.perf_counter()
    pending = []
    dev = None
    pipe = None

    def emit(out, air):
        nonlocal count
        if sink is not None:
            sink(out)
        trace.append(air)
        count += 1

    def flush():
        if pipe is not None:
            pipe.finish(emit)
            return
        if not pending:
            return
        batch = _as_device_batch(np.stack(pending), dev)
        out, air = dehaze_batch(batch, params)
        out_h = out.cpu().numpy()
        air_h = air.cpu().numpy()
        for i in range(len(pending)):
            emit(out_h[i], air_h[i].copy())
        pending.clear()

    try:
        it = iter(frames)
        index = -1
        while True:
            index += 1
            try:
                frame = next(it)
            except StopIteration:
                break
            except BaseException:
                flush()  # frames before a failing source (e.g. a truncated stream) still reach the sink
                raise
            try:
                frame = check_u8_frame(frame, name=f"frame {index}")
                if not isinstance(frame, np.ndarray):
                    frame = frame.cpu().numpy()
                if expected_shape is None:
                    expected_shape = frame.shape
                    dev = _device()
                    per = frame.nbytes
                    limit = max(1, min(_STREAM_BATCH_MAX, _STREAM_BATCH_BYTES // max(per, 1)))
                    if _native_ok(params, frame.shape[0], frame.shape[1]):
                        pipe = _acquire_pipe(devs if devs is not None else [dev], params, frame.shape, lam, n_hint)
                    elif devs is not None or lam is not None:
                        raise ValueError("devices= / stabilise= need a call the batched native pipeline covers "
                                         "(see _native_ok)")
                elif frame.shape != expected_shape:
                    raise ValueError(
                        f"frame {index} has size {frame.shape[1]}x{frame.shape[0]}, "
                        f"expected {expected_shape[1]}x{expected_shape[0]}"
                    )
            except ValueError:
                flush()
                raise
            if pipe is not None:
                pipe.put(frame, emit, persistent=persistent)
                continue
            pending.append(frame)
            if len(pending) >= limit:
                flush()
        flush()
    finally:
        if pipe is not None:
            pipe.busy = False  # back to the thread's cache (see _acquire_pipe)

    wall = time.perf_counter() - start
    fps = count / wall if wall > 0 and count else 0.0
    return StreamStats(frame_count=count, wall_time=wall, fps=fps, airlight_trace=trace)
