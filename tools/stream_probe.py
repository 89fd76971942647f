"""Throughput of the reference-shaped host API (process_stream over numpy frames, a sink
per frame) against dehaze_host_batch on the same frames."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_16609_b200 import DehazeParams, dehaze_host_batch, process_stream
from paper_2512_16609_b200.synthetic import make_frames

n = int(os.environ.get("N", 300))
frames_t = make_frames("c3", frames=n, device="cuda").cpu()
frames = [f.numpy() for f in frames_t]
for name, p in (("native", DehazeParams(resize_to=None)), ("default-resize", DehazeParams())):
    got = []
    process_stream(frames[:8], p, sink=got.append)  # warm-up
    got.clear()
    t0 = time.perf_counter()
    st = process_stream(frames, p, sink=got.append)
    el = time.perf_counter() - t0
    print(f"process_stream {name}: {n / el:.0f} fps, {n * 1920 * 1080 / el / 1e6:.0f} MP/s ({el * 1e3:.1f} ms)")
    pin = frames_t.pin_memory()
    dehaze_host_batch(pin, p)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dehaze_host_batch(pin, p)
    el = time.perf_counter() - t0
    print(f"dehaze_host_batch {name}: {n / el:.0f} fps ({el * 1e3:.1f} ms)")

# raw RGB24 streams: reader + process_stream + writer vs the pinned-staging path
import io

from paper_2512_16609_b200.frameio import StreamHeader, dehaze_raw_stream, read_raw_frames, write_raw_frame

raw = b"".join(f.tobytes() for f in frames)
hdr = StreamHeader(width=1920, height=1080)
for name, p in (("native", DehazeParams(resize_to=None)), ("default-resize", DehazeParams())):
    dst = io.BytesIO()
    t0 = time.perf_counter()
    process_stream(read_raw_frames(io.BytesIO(raw), hdr), p, sink=lambda f: write_raw_frame(dst, f))
    el = time.perf_counter() - t0
    dst2 = io.BytesIO()
    t0 = time.perf_counter()
    dehaze_raw_stream(io.BytesIO(raw), dst2, hdr, p)
    el2 = time.perf_counter() - t0
    print(f"raw stream {name}: reader+process_stream+writer {n / el:.0f} fps, dehaze_raw_stream {n / el2:.0f} fps,"
          f" same bytes {dst.getvalue() == dst2.getvalue()}")
