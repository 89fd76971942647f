"""Sweep (streams, chunk) for the CUDA-graph-captured chunked pipeline on the C3 workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import FrameEngine, GraphedPipeline
from paper_2512_16609_b200.synthetic import Scene

dev = torch.device("cuda", 0)
n, H, W = int(os.environ.get("N", 300)), 1080, 1920
scene = Scene(W, H, 3000, dev)
frames = torch.stack([scene.hazy_u8(f, 3000 + f, 0.6, (0.85, 0.87, 0.9)) for f in range(n)])
params = DehazeParams(resize_to=None, white_balance=bool(int(os.environ.get("BAL", "0"))))
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


CASES = [tuple(int(v) for v in c.split("x")) for c in os.environ.get("CASES", "").split(",") if c] or \
    [(1, n), (2, 4), (2, 8), (2, 16), (2, 32), (3, 4), (3, 8), (4, 4), (4, 8)]
for S, C in CASES:
    gp = GraphedPipeline(frames, params, streams=S, chunk=C)
    ms = bench(gp.replay)
    ok = torch.equal(gp.out, ref_out) and torch.equal(gp.airlight, ref_air)
    print(f"graph streams={S} chunk={C} ms={ms:.4f} exact={ok}", flush=True)
    del gp
    torch.cuda.empty_cache()
