"""Raw RGB24 frame streams (reference frameio.py:215-291) and a GPU streaming path.

The byte stream is headerless: frames of width*height*3 interleaved RGB bytes back
to back; a ``StreamHeader`` describes it out of band.  ``read_raw_frames`` /
``write_raw_frame`` keep the reference's contract (errors, messages, the offset of
a truncated frame); ``dehaze_raw_stream`` is the B200 path for the same job as the
reference CLI's ``process_stream(read_raw_frames(...), sink=write_raw_frame)``: frames
are read with ``readinto`` straight into pinned staging buffers and written back
from pinned output buffers, so no per-frame host array is ever allocated.

Image codecs (PPM, PNG, image directories) stay out of scope.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .validation import check_u8_frame


class CodecError(ValueError):
    """Base of the frame I/O errors (reference frameio.py:25)."""


class RawStreamError(CodecError):
    pass


class RawStreamTruncated(RawStreamError):
    """The stream ended inside a frame; ``offset`` is the byte where that frame began."""

    def __init__(self, message, offset):
        super().__init__(message)
        self.offset = offset


@dataclass(frozen=True)
class StreamHeader:
    """Geometry of a raw RGB24 stream; frame_count=None reads until the stream ends."""

    width: int
    height: int
    frame_count: int = None

    def __post_init__(self):
        for name in ("width", "height"):
            v = getattr(self, name)
            if int(v) != v or v < 1:
                raise RawStreamError(f"invalid stream {name} {v}")
        c = self.frame_count
        if c is not None and (int(c) != c or c < 0):
            raise RawStreamError(f"invalid frame count {c}")

    @property
    def frame_bytes(self):
        return 3 * self.width * self.height


def _fill(stream, view):
    """Read into ``view`` until it is full or the stream ends; returns the bytes read."""
    got = 0
    n = len(view)
    readinto = getattr(stream, "readinto", None)
    while got < n:
        if readinto is not None:
            try:
                k = readinto(view[got:])
            except NotImplementedError:  # e.g. an io.RawIOBase that only overrides read()
                readinto = None
                continue
            k = 0 if k is None else k
        else:
            chunk = stream.read(n - got)
            k = len(chunk)
            view[got:got + k] = chunk
        if k == 0:
            break
        got += k
    return got


def _short_read(header, got, offset, produced):
    """The error for a frame that came back with ``got`` < frame_bytes bytes (None: clean end)."""
    if got == 0:
        if header.frame_count is not None and produced < header.frame_count:
            return RawStreamTruncated(
                f"stream ended at byte offset {offset} after {produced} frames, expected {header.frame_count}",
                offset)
        return None
    return RawStreamTruncated(
        f"truncated frame at byte offset {offset}: got {got} of {header.frame_bytes} bytes", offset)


def read_raw_frames(stream, header):
    """Yield (height, width, 3) uint8 frames from a raw RGB24 binary stream.

    Raises RawStreamTruncated when the stream ends inside a frame (or before a
    declared frame_count); its ``offset`` is the byte where the broken frame began.
    """
    size = header.frame_bytes
    produced = 0
    while header.frame_count is None or produced < header.frame_count:
        frame = np.empty((header.height, header.width, 3), dtype=np.uint8)
        got = _fill(stream, memoryview(frame).cast("B"))
        if got < size:
            err = _short_read(header, got, produced * size, produced)
            if err is None:
                return
            raise err
        yield frame
        produced += 1


def write_raw_frame(stream, frame):
    """Append one frame (validated like every other frame input) to a raw RGB24 stream."""
    frame = check_u8_frame(frame)
    stream.write(memoryview(np.ascontiguousarray(frame)).cast("B"))


def dehaze_raw_stream(src, dst, header, params=None):
    """Dehaze a raw RGB24 stream into another, in order, on the GPU.

    Same result as ``process_stream(read_raw_frames(src, header), params,
    sink=lambda f: write_raw_frame(dst, f))`` (frames before a truncated one are
    written before RawStreamTruncated is raised), with reads and writes going
    through the pinned staging of the pipelined batches.  Returns StreamStats.
    """
    from .pipeline import DehazeParams, StreamStats, _StreamPipe, _device, _native_ok, process_stream

    if params is None:
        params = DehazeParams()
    params.validate()
    H, W = header.height, header.width
    if not _native_ok(params, H, W):
        return process_stream(read_raw_frames(src, header), params, sink=lambda f: write_raw_frame(dst, f))

    start = time.perf_counter()
    trace = []
    count = 0

    def emit(out, air):
        nonlocal count
        dst.write(out)
        trace.append(air)
        count += 1

    pipe = _StreamPipe([_device()], params, (H, W, 3), fresh=False)
    size = header.frame_bytes
    produced = 0
    err = None
    while header.frame_count is None or produced < header.frame_count:
        view = pipe.next_input(emit)
        got = _fill(src, memoryview(view.numpy()).cast("B"))
        if got < size:
            err = _short_read(header, got, produced * size, produced)
            break
        pipe.commit(emit)
        produced += 1
    pipe.finish(emit)
    if err is not None:
        raise err
    wall = time.perf_counter() - start
    return StreamStats(frame_count=count, wall_time=wall, fps=count / wall if wall > 0 and count else 0.0,
                       airlight_trace=trace)
