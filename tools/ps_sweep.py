"""process_stream throughput vs the pipelined batch size and slot count (C3 / C4 frames)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams, process_stream
from paper_2512_16609_b200 import pipeline as pl
from paper_2512_16609_b200.synthetic import make_frames

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
nfr = int(sys.argv[2]) if len(sys.argv) > 2 else 300
frames = [f.numpy().copy() for f in make_frames(cfg, frames=nfr, device="cuda").cpu()]
p = DehazeParams(resize_to=None, white_balance=True if cfg == "c4" else None)
npx = frames[0].shape[0] * frames[0].shape[1]
for slots in (3, 4):
    for mb in (12, 24, 48, 96):
        pl._PIPE_SLOTS = slots
        pl._PIPE_BATCH_BYTES = mb << 20
        process_stream(frames, p, sink=lambda o: None)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            process_stream(frames, p, sink=lambda o: None)
            ts.append(time.perf_counter() - t0)
        best, med = min(ts), sorted(ts)[len(ts) // 2]
        print(f"{cfg} slots={slots} batch={mb} MiB: best {nfr * npx / best / 1e6:.0f} MP/s, median {nfr * npx / med / 1e6:.0f} MP/s", flush=True)
