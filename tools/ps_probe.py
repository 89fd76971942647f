"""process_stream per-call time for small clips (bench e2e.process_stream legs), A/B of
the native copy threads (DHZ_HOST_COPY=0 falls back to torch copies)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_16609_b200 import DehazeParams, process_stream, pipeline
from paper_2512_16609_b200.synthetic import make_frames

for cfg, p, n in [("c1", DehazeParams(resize_to=None), 1), ("c2", DehazeParams.for_image(guided_radius=30), 1),
                  ("c3", DehazeParams(resize_to=None), 32)]:
    frames = [f.numpy() for f in make_frames(cfg, frames=n, device="cuda").cpu()]
    ts = []
    for it in range(6):
        t0 = time.perf_counter()
        process_stream(frames, p, sink=lambda o: None)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(cfg, n, "frames; ms per call:", " ".join(f"{t:.2f}" for t in ts), flush=True)
