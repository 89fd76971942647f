"""Device-side batch engine: owns workspaces and launches the fused frame pipeline.

Frames live in HBM as one contiguous uint8 tensor (n, H, W, 3); one call of
``FrameEngine.run`` enqueues the whole batch (K1 dark -> K2..K4 top-K select +
airlight -> K5 LUT -> K6 recover) on a CUDA stream through the
C ABI.  Nothing here touches pixel data on the CPU.
"""

from __future__ import annotations

import ctypes
import math
import threading

import torch

from . import _native
from .quant import device_thresholds


MAX_FRAMES_PER_CALL = 65535  # abi.cu kMaxFrames (frames ride grid.y / grid.z)


def top_k(npx: int, top_fraction: float) -> int:
    """estimation.py:72 — K = max(1, floor(top_fraction * n)), Python float arithmetic."""
    return max(1, math.floor(top_fraction * npx))


def _check_buffer(t, name, shape, dtype, dev):
    """Caller-supplied output buffers: the ABI writes through raw pointers."""
    if not isinstance(t, torch.Tensor) or t.device != dev or t.dtype != dtype or tuple(t.shape) != tuple(shape) \
            or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)} on {dev}, got "
                         f"{tuple(getattr(t, 'shape', ()))} {getattr(t, 'dtype', type(t))} "
                         f"on {getattr(t, 'device', '?')}")


def native_params(params, npx: int, thresholds: torch.Tensor) -> _native.DhzParams:
    p = _native.DhzParams()
    p.mode = 1 if params.mode == "image" else 0
    p.patch_radius = int(params.patch_radius)
    p.top_k = top_k(npx, params.top_fraction)
    p.alpha = float(params.alpha)
    p.omega = float(params.omega)
    p.t_min = float(params.t_min)
    p.guided_radius = int(params.guided_radius)
    p.balance = 1 if params.balance_enabled() else 0
    p.guided_eps = float(params.guided_eps)
    p.gamma = float(params.gamma)
    p.thresholds = thresholds.data_ptr()
    return p


class FrameEngine:
    """Runs the fused u8 pipeline over device-resident frame batches on one GPU."""

    def __init__(self, device=None):
        self.lib = _native.lib()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self._ws = None
        self._lock = threading.Lock()
        # the workspace is reused by every run: a run enqueued on another stream
        # waits for the previous run's kernels (event recorded after each run)
        self._last = None  # (cuda stream handle, torch.cuda.Event)

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.device)
        return self._ws

    def _order_after_last(self, st):
        last = self._last
        if last is None or last[0] == st.cuda_stream:
            return
        if torch.cuda.is_current_stream_capturing():
            return  # inside a graph capture the caller orders the captured work
        st.wait_event(last[1])

    def _mark_done(self, st):
        if torch.cuda.is_current_stream_capturing():
            self._last = None
            return
        ev = torch.cuda.Event()
        ev.record(st)
        self._last = (st.cuda_stream, ev)

    def _maps(self, ws, n, h, w, H, W, p, resize, st):
        """Copies of the dark map and selected indices left in the workspace (on ``st``)."""
        k = p.top_k
        with torch.cuda.stream(st):
            if resize:
                off = (ctypes.c_int64 * 5)()
                _native.check(self.lib.dhz_frames_resize_u8_layout(n, h, w, H, W, ctypes.byref(p), off),
                              "dhz_frames_resize_u8_layout")
                maps = {"dark_f64": ws[off[0]: off[0] + off[1] * n].view(torch.float64).view(n, H, W).clone()}
            else:
                off = self.layout(n, H, W, p)
                dark_fs = off[1]
                maps = {"dark_u8": ws[off[0]: off[0] + dark_fs * n].view(n, dark_fs)[:, : H * W]
                        .reshape(n, H, W).clone()}
            maps["selected"] = ws[off[2]: off[2] + 4 * n * k].view(torch.int32).view(n, k).clone()
        return maps

    def layout(self, n, H, W, p):
        off = (ctypes.c_int64 * 5)()
        _native.check(self.lib.dhz_frames_u8_layout(n, H, W, ctypes.byref(p), off), "dhz_frames_u8_layout")
        return list(off)

    def _ws_bytes(self, n, h, w, H, W, p):
        if (H, W) != (h, w):
            nbytes = self.lib.dhz_frames_resize_u8_workspace(n, h, w, H, W, ctypes.byref(p))
        else:
            nbytes = self.lib.dhz_frames_u8_workspace(n, H, W, ctypes.byref(p))
        if nbytes == 0:
            _native.check(_native.DHZ_E_INVALID, "workspace query")
        return nbytes

    def phase_airlight(self, frames, params, airlight=None, stream=None):
        """First half of the pipeline (dark channel + top-K select): the (n, 3) airlight."""
        n, h, w, _ = frames.shape
        H, W = self.working_size(params, h, w)
        dev = frames.device
        if airlight is None:
            airlight = torch.empty((n, 3), dtype=torch.float64, device=dev)
        else:
            _check_buffer(airlight, "airlight", (n, 3), torch.float64, dev)
        if n == 0:
            return airlight
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        p = native_params(params, H * W, device_thresholds(params.gamma, dev))
        with self._lock, torch.cuda.device(dev):
            self._order_after_last(st)
            ws = self.workspace(self._ws_bytes(n, h, w, H, W, p))
            if (H, W) != (h, w):
                rc = self.lib.dhz_frames_resize_u8_airlight(frames.data_ptr(), 3 * h * w, n, h, w, H, W,
                                                            ctypes.byref(p), airlight.data_ptr(), ws.data_ptr(),
                                                            ws.numel(), st.cuda_stream)
            else:
                rc = self.lib.dhz_frames_u8_airlight(frames.data_ptr(), 3 * H * W, n, H, W, ctypes.byref(p),
                                                     airlight.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)
            _native.check(rc, "dhz_frames_*_airlight")
            self._mark_done(st)
        return airlight

    def phase_recover(self, frames, params, airlight, out=None, stream=None):
        """Second half (transmission [+ guided filter], recovery, output) from a given airlight."""
        n, h, w, _ = frames.shape
        H, W = self.working_size(params, h, w)
        dev = frames.device
        _check_buffer(airlight, "airlight", (n, 3), torch.float64, dev)
        if out is None:
            out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=dev)
        else:
            _check_buffer(out, "out", (n, H, W, 3), torch.uint8, dev)
        if n == 0:
            return out
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        p = native_params(params, H * W, device_thresholds(params.gamma, dev))
        with self._lock, torch.cuda.device(dev):
            self._order_after_last(st)
            ws = self.workspace(self._ws_bytes(n, h, w, H, W, p))
            if (H, W) != (h, w):
                rc = self.lib.dhz_frames_resize_u8_recover(frames.data_ptr(), 3 * h * w, n, h, w, H, W,
                                                           ctypes.byref(p), airlight.data_ptr(), out.data_ptr(),
                                                           3 * H * W, ws.data_ptr(), ws.numel(), st.cuda_stream)
            else:
                rc = self.lib.dhz_frames_u8_recover(frames.data_ptr(), 3 * H * W, n, H, W, ctypes.byref(p),
                                                    airlight.data_ptr(), out.data_ptr(), 3 * H * W, ws.data_ptr(),
                                                    ws.numel(), st.cuda_stream)
            _native.check(rc, "dhz_frames_*_recover")
            self._mark_done(st)
        return out

    @staticmethod
    def working_size(params, H, W):
        """(height, width) the pipeline runs at: resize_to, or the native size."""
        if params.resize_to is None:
            return H, W
        rw, rh = (int(v) for v in params.resize_to)
        return rh, rw

    def run(self, frames: torch.Tensor, params, out: torch.Tensor | None = None,
            airlight: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None,
            keep_maps: bool = False, events=None, stabilise: float | None = None,
            carry: torch.Tensor | None = None):
        """Dehaze ``frames`` (n, H, W, 3) uint8 CUDA, C-contiguous.

        Frames are first resized to ``params.resize_to`` when that differs from
        their size (video mode, dhz_frames_resize_u8).  Returns (out uint8
        (n, H', W', 3), airlight float64 (n, 3)) as CUDA tensors, plus a dict of
        device maps when ``keep_maps`` (dark map — u8 at native size, float64
        after a resize — and the selected indices).

        ``stabilise=lam`` (opt-in, NOT reference behaviour): the frames' airlight
        trace is smoothed by the recurrence A'_f = lam A'_{f-1} + (1 - lam) A_f
        (dhz_ema_airlight; A'_-1 = ``carry`` (3,) when given) between the airlight
        and the recovery halves of the pipeline; the returned airlight is A'.
        """
        if frames.dim() != 4 or frames.shape[-1] != 3 or frames.dtype != torch.uint8:
            raise ValueError(f"frames must be (n, H, W, 3) uint8, got {tuple(frames.shape)} {frames.dtype}")
        if not frames.is_cuda:
            raise ValueError("frames must be a CUDA tensor")
        frames = frames.contiguous()
        n, h, w, _ = frames.shape
        H, W = self.working_size(params, h, w)
        resize = (H, W) != (h, w)
        dev = frames.device
        thr = device_thresholds(params.gamma, dev)
        p = native_params(params, H * W, thr)
        if out is None:
            out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=dev)
        else:
            _check_buffer(out, "out", (n, H, W, 3), torch.uint8, dev)
        if airlight is None:
            airlight = torch.empty((n, 3), dtype=torch.float64, device=dev)
        else:
            _check_buffer(airlight, "airlight", (n, 3), torch.float64, dev)
        if n == 0:
            return (out, airlight, {}) if keep_maps else (out, airlight)
        if n > MAX_FRAMES_PER_CALL and not keep_maps:  # the library takes <= 65535 frames per call
            for lo in range(0, n, MAX_FRAMES_PER_CALL):
                hi = min(n, lo + MAX_FRAMES_PER_CALL)
                self.run(frames[lo:hi], params, out=out[lo:hi], airlight=airlight[lo:hi], stream=stream,
                         stabilise=stabilise, carry=carry if lo == 0 else airlight[lo - 1])
            return out, airlight
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        if stabilise is not None:
            if keep_maps or events is not None:
                raise ValueError("stabilise= runs the two-phase path (no maps / stage events)")
            raw = self.phase_airlight(frames, params, stream=st)
            ema_airlight(raw, stabilise, carry=carry, out=airlight, stream=st)
            self.phase_recover(frames, params, airlight, out=out, stream=st)
            return out, airlight
        ev_arr = None
        if events is not None:
            # torch creates events lazily: record once so each has a handle, then
            # let the library re-record them between the fused stages.
            for ev in events:
                ev.record(st)
            ev_arr = (ctypes.c_void_p * len(events))(*[ev.cuda_event for ev in events])
        with self._lock, torch.cuda.device(dev):
            self._order_after_last(st)
            if resize:
                nbytes = self.lib.dhz_frames_resize_u8_workspace(n, h, w, H, W, ctypes.byref(p))
                if nbytes == 0:
                    _native.check(_native.DHZ_E_INVALID, "dhz_frames_resize_u8_workspace")
                ws = self.workspace(nbytes)
                rc = self.lib.dhz_frames_resize_u8(
                    frames.data_ptr(), 3 * h * w, n, h, w, H, W, ctypes.byref(p), out.data_ptr(), 3 * H * W,
                    airlight.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream, ev_arr)
                _native.check(rc, "dhz_frames_resize_u8")
            else:
                nbytes = self.lib.dhz_frames_u8_workspace(n, H, W, ctypes.byref(p))
                if nbytes == 0:
                    _native.check(_native.DHZ_E_INVALID, "dhz_frames_u8_workspace")
                ws = self.workspace(nbytes)
                rc = self.lib.dhz_frames_u8(
                    frames.data_ptr(), 3 * H * W, n, H, W, ctypes.byref(p), out.data_ptr(), 3 * H * W,
                    airlight.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream, ev_arr)
                _native.check(rc, "dhz_frames_u8")
            maps = self._maps(ws, n, h, w, H, W, p, resize, st) if keep_maps else None
            self._mark_done(st)
        if keep_maps:
            return out, airlight, maps
        return out, airlight


def ema_airlight(trace: torch.Tensor, lam: float, carry: torch.Tensor | None = None,
                 out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Opt-in temporal stabilisation of an (n, 3) float64 CUDA airlight trace
    (dhz_ema_airlight): A'_f = lam A'_{f-1} + (1 - lam) A_f, each product and sum
    rounded once; A'_-1 = ``carry`` when given, else A'_0 = A_0.  NOT reference
    behaviour (reference SPEC.md:267 lists temporal smoothing as a non-goal)."""
    lam = float(lam)
    if not 0.0 <= lam < 1.0:
        raise ValueError(f"stabilise must lie in [0, 1), got {lam}")
    n = int(trace.shape[0])
    dev = trace.device
    trace = trace.contiguous()
    if out is None:
        out = torch.empty_like(trace)
    if carry is not None:
        carry = carry.to(device=dev, dtype=torch.float64).contiguous()
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        rc = _native.lib().dhz_ema_airlight(trace.data_ptr(), n, lam, carry.data_ptr() if carry is not None else None,
                                            out.data_ptr(), st.cuda_stream)
    _native.check(rc, "dhz_ema_airlight")
    return out


class DeviceGroup:
    """Several GPUs (or several shards on one GPU) behind dhz_comm_init: one engine and
    one stream per shard, and the airlight all-gather between them."""

    def __init__(self, devices):
        devs = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
        if not devs:
            raise ValueError("devices must name at least one CUDA device")
        for d in devs:
            if d.type != "cuda":
                raise ValueError(f"devices must be CUDA devices, got {d}")
        self.devices = [torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())
                        for d in devs]
        self.lib = _native.lib()
        self.engines = [FrameEngine(d) for d in self.devices]
        self.streams = [torch.cuda.Stream(d) for d in self.devices]
        ids = (ctypes.c_int * len(self.devices))(*[d.index for d in self.devices])
        h = ctypes.c_void_p()
        _native.check(self.lib.dhz_comm_init(len(self.devices), ids, ctypes.byref(h)), "dhz_comm_init")
        self._comm = h

    def __del__(self):
        if getattr(self, "_comm", None):
            try:
                self.lib.dhz_comm_destroy(self._comm)
            except Exception:
                pass
            self._comm = None

    def allgather_airlight(self, blocks, counts):
        """blocks[d]: (counts[d], 3) float64 on device d -> per device the (sum, 3) trace."""
        total = sum(counts)
        k = len(self.devices)
        recv = [torch.empty((total, 3), dtype=torch.float64, device=d) for d in self.devices]
        send_p = (ctypes.c_void_p * k)(*[b.data_ptr() for b in blocks])
        recv_p = (ctypes.c_void_p * k)(*[r.data_ptr() for r in recv])
        cnt = (ctypes.c_int * k)(*counts)
        sts = (ctypes.c_void_p * k)(*[s.cuda_stream for s in self.streams])
        _native.check(self.lib.dhz_allgather_airlight(self._comm, send_p, cnt, recv_p, sts), "dhz_allgather_airlight")
        return recv

    def run(self, frames: torch.Tensor, params, out: torch.Tensor | None = None, stabilise: float | None = None):
        """Dehaze a (n, H, W, 3) uint8 batch (host or any device) sharded by frame over the
        group: contiguous blocks (shard_range), each dehazed on its device; the airlight
        trace is all-gathered (every device holds it in frame order) and, with
        ``stabilise``, smoothed on every device before the recovery half.  Returns
        (out, airlight) on ``frames``' device (outputs copied back in frame order)."""
        from .distributed import shard_range

        n, h, w = (int(v) for v in frames.shape[:3])
        H, W = FrameEngine.working_size(params, h, w)
        home = frames.device if frames.is_cuda else self.devices[0]
        if out is None:
            out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=home)
        airlight = torch.empty((n, 3), dtype=torch.float64, device=home)
        if n == 0:
            return out, airlight
        k = len(self.devices)
        ranges = [shard_range(n, i, k) for i in range(k)]
        cur = torch.cuda.current_stream(home) if frames.is_cuda else None
        locals_ = []
        for i, (lo, hi) in enumerate(ranges):
            dev, st = self.devices[i], self.streams[i]
            if cur is not None:
                st.wait_stream(cur)
            with torch.cuda.stream(st):
                src = frames[lo:hi]
                f_d = src if (src.is_cuda and src.device == dev) else src.to(dev, non_blocking=True)
                raw = self.engines[i].phase_airlight(f_d, params, stream=st) if hi > lo else \
                    torch.empty((0, 3), dtype=torch.float64, device=dev)
            locals_.append((f_d, raw))
        traces = self.allgather_airlight([r for _, r in locals_], [hi - lo for lo, hi in ranges])
        for i, (lo, hi) in enumerate(ranges):
            dev, st = self.devices[i], self.streams[i]
            f_d, _ = locals_[i]
            with torch.cuda.stream(st):
                trace = traces[i]
                if stabilise is not None:
                    trace = ema_airlight(trace, stabilise, stream=st)
                if i == 0:
                    airlight.copy_(trace, non_blocking=True)
                if hi > lo:
                    mine = trace[lo:hi]
                    o_d = self.engines[i].phase_recover(f_d, params, mine, stream=st)
                    out[lo:hi].copy_(o_d, non_blocking=True)
        if cur is not None:
            for st in self.streams:
                cur.wait_stream(st)
        else:
            for st in self.streams:
                st.synchronize()
        return out, airlight


class StreamedEngine:
    """Chunks a device batch over several CUDA streams (one workspace each).

    Consecutive chunks run on different streams, so the dark-channel pass of
    one chunk (HBM/ALU heavy) overlaps the LUT recovery pass of another
    (shared-memory bound), and a chunk's frames are still L2-resident when its
    recovery pass re-reads them.
    """

    def __init__(self, device, streams=2):
        self.device = torch.device(device)
        self.engines = [FrameEngine(self.device) for _ in range(streams)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(streams)]

    def run(self, frames, params, out=None, airlight=None, chunk=16):
        n, h, w = (int(v) for v in frames.shape[:3])
        if out is None:
            H, W = FrameEngine.working_size(params, h, w)
            out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=frames.device)
        if airlight is None:
            airlight = torch.empty((n, 3), dtype=torch.float64, device=frames.device)
        cur = torch.cuda.current_stream(self.device)
        for st in self.streams:
            st.wait_stream(cur)
        for c, lo in enumerate(range(0, n, chunk)):
            k = c % len(self.streams)
            hi = min(n, lo + chunk)
            self.engines[k].run(frames[lo:hi], params, out=out[lo:hi], airlight=airlight[lo:hi],
                                stream=self.streams[k])
        for st in self.streams:
            cur.wait_stream(st)
        return out, airlight


class GraphedPipeline:
    """A fixed (frames, params) batch captured once as a CUDA graph and replayed.

    With ``streams > 1`` the batch is cut into ``chunk``-frame pieces spread over
    the streams (StreamedEngine), so one chunk's dark-channel pass (ALU/HBM)
    overlaps another chunk's LUT pass (shared-memory bound) and the recovery pass
    finds its chunk's frames in L2; the graph removes the per-launch host cost
    that would otherwise dominate small chunks.  Inputs/outputs are the tensors
    given at construction (update ``frames`` in place between replays).  With
    ``streams == 1``, ``events`` (DHZ_N_EVENTS timing events) are recorded by every
    replay at the stage boundaries.
    """

    def __init__(self, frames, params, out=None, airlight=None, streams=2, chunk=8, events=None):
        self.frames = frames
        self.params = params
        n, h, w = (int(v) for v in frames.shape[:3])
        H, W = FrameEngine.working_size(params, h, w)
        self.out = out if out is not None else torch.empty((n, H, W, 3), dtype=torch.uint8, device=frames.device)
        self.airlight = airlight if airlight is not None else torch.empty(
            (n, 3), dtype=torch.float64, device=frames.device)
        self.streams = streams
        self.chunk = chunk
        if streams > 1:
            self._eng = StreamedEngine(frames.device, streams)
            run = lambda: self._eng.run(self.frames, params, out=self.out, airlight=self.airlight, chunk=chunk)  # noqa: E731
        else:
            self._eng = FrameEngine(frames.device)
            run = lambda ev=None: self._eng.run(self.frames, params, out=self.out, airlight=self.airlight,  # noqa: E731
                                                events=ev)
        run()  # eager warm-up: workspaces, thresholds, kernel attributes
        torch.cuda.synchronize(frames.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            # stage events (single-stream only) are captured as event-record nodes:
            # every replay re-timestamps them
            run(events) if streams == 1 and events is not None else run()
        torch.cuda.synchronize(frames.device)

    def replay(self):
        self.graph.replay()
        return self.out, self.airlight


_engines: dict = {}
_engines_lock = threading.Lock()


def engine_for(device=None) -> FrameEngine:
    """Per-(device, thread) engine so concurrent callers never share a workspace."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    key = (device.index, threading.get_ident())
    with _engines_lock:
        eng = _engines.get(key)
        if eng is None:
            eng = FrameEngine(device)
            _engines[key] = eng
    return eng
