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
