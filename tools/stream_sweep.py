"""Sweep (streams, chunk) for the chunked multi-stream engine on the C3 workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import FrameEngine, StreamedEngine
from paper_2512_16609_b200.synthetic import Scene

dev = torch.device("cuda", 0)
n, H, W = int(os.environ.get("N", 300)), 1080, 1920
scene = Scene(W, H, 3000, dev)
frames = torch.stack([scene.hazy_u8(f, 3000 + f, 0.6, (0.85, 0.87, 0.9)) for f in range(n)])
params = DehazeParams(resize_to=None)
ref_out, ref_air = FrameEngine(dev).run(frames, params)
torch.cuda.synchronize()


def bench(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


eng = FrameEngine(dev)
out = torch.empty_like(frames)
air = torch.empty((n, 3), dtype=torch.float64, device=dev)
print("single", round(bench(lambda: eng.run(frames, params, out=out, airlight=air)), 4), flush=True)
for S, C in [(2, 8), (2, 16), (2, 32), (3, 8), (3, 16), (4, 8), (4, 16), (6, 8)]:
    se = StreamedEngine(dev, S)
    ms = bench(lambda: se.run(frames, params, out=out, airlight=air, chunk=C))
    ok = torch.equal(out, ref_out) and torch.equal(air, ref_air)
    print(f"streams={S} chunk={C} ms={ms:.4f} exact={ok}", flush=True)
