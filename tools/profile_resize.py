"""Small driver for ncu: the batched default-resize path on 1080p frames."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import engine_for
from paper_2512_16609_b200.synthetic import Scene

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=32)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--balance", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
scene = Scene(1920, 1080, 3000, dev)
frames = torch.stack([scene.hazy_u8(f, 3000 + f, 0.6, (0.85, 0.87, 0.9)) for f in range(a.frames)])
params = DehazeParams(white_balance=a.balance)
eng = engine_for(dev)
for _ in range(a.iters):
    out, air = eng.run(frames, params)
torch.cuda.synchronize()
print("ok", out.shape, air[0].tolist())
