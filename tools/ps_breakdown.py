"""Where process_stream's wall time goes (C3/C4 frames): per-method wall-time totals of
_StreamPipe, raw host-copy bandwidth of the box, for sizing the copy scheme."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_16609_b200 import DehazeParams, process_stream
from paper_2512_16609_b200 import pipeline as pl
from paper_2512_16609_b200.synthetic import make_frames

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
nfr = int(sys.argv[2]) if len(sys.argv) > 2 else 120
frames = [f.numpy().copy() for f in make_frames(cfg, frames=nfr, device="cuda").cpu()]
p = DehazeParams(resize_to=None, white_balance=(cfg == "c4") or None)
nb = frames[0].nbytes

# raw copy bandwidth: pageable -> pinned, k threads, one frame per job
pin = torch.empty((16,) + frames[0].shape, dtype=torch.uint8, pin_memory=True)
from concurrent.futures import ThreadPoolExecutor
for k in (1, 2, 4, 8, 16):
    ex = ThreadPoolExecutor(k)
    jobs = list(range(16))
    def cp(i):
        pin[i].copy_(torch.from_numpy(frames[i % len(frames)]))
    list(ex.map(cp, jobs))
    t0 = time.perf_counter()
    for _ in range(5):
        list(ex.map(cp, jobs))
    el = (time.perf_counter() - t0) / 5
    print(f"copy {k:2d} threads: {16 * nb / el / 1e9:6.1f} GB/s ({el * 1e3 / 16:.3f} ms/frame)", flush=True)
    ex.shutdown()

tot = {}
def wrap(name):
    f = getattr(pl._StreamPipe, name)
    def g(self, *a, **kw):
        t0 = time.perf_counter()
        try:
            return f(self, *a, **kw)
        finally:
            tot[name] = tot.get(name, 0.0) + time.perf_counter() - t0
    setattr(pl._StreamPipe, name, g)
for nm in ("put", "submit", "drain", "finish", "next_input"):
    wrap(nm)
process_stream(frames[:8], p, sink=lambda o: None)
for rep in range(3):
    tot.clear()
    t0 = time.perf_counter()
    st = process_stream(frames, p, sink=lambda o: None)
    el = time.perf_counter() - t0
    print(f"{cfg} {nfr} frames: {el * 1e3:.1f} ms ({nfr * nb / 3 / el / 1e6:.0f} MP/s) "
          + " ".join(f"{k}={v * 1e3:.1f}" for k, v in sorted(tot.items())), flush=True)
