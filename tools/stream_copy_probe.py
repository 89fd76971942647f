"""process_stream host-copy variants on C3 frames: copy threads on/off for the input
staging and the fresh output arrays (pipeline._COPY_THREADS, _par_copy)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2512_16609_b200 import DehazeParams, process_stream, pipeline
from paper_2512_16609_b200.synthetic import make_frames

n = int(os.environ.get("N", 300))
frames_t = make_frames("c3", frames=n, device="cuda").cpu()
frames = [f.numpy() for f in frames_t]
p = DehazeParams(resize_to=None)
orig_par = pipeline._par_copy
for threads in (1, 2, 4, 8, 16):
    pipeline._COPY_THREADS = threads
    pipeline._copy_pool = None
    for keep in (False, True):
        got = []
        sink = got.append if keep else (lambda o: None)
        process_stream(frames[:16], p, sink=sink)
        got.clear()
        t0 = time.perf_counter()
        process_stream(frames, p, sink=sink)
        el = time.perf_counter() - t0
        print(f"threads {threads:2d} sink keeps outputs {keep}: {n / el:6.0f} fps {n * 2.0736 / el:7.0f} MP/s", flush=True)
# page-fault cost of fresh arrays
t0 = time.perf_counter()
for _ in range(100):
    a = np.empty((1080, 1920, 3), np.uint8); a[...] = 1
print("fresh 6.2 MB array + fill: %.3f ms" % ((time.perf_counter() - t0) * 10))
b = np.empty((1080, 1920, 3), np.uint8); b[...] = 0
t0 = time.perf_counter()
for _ in range(100):
    b[...] = 1
print("reused array fill: %.3f ms" % ((time.perf_counter() - t0) * 10))
