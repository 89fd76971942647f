"""Small driver for ncu: runs the fused pipeline (video, or image mode with --image R) a few times."""
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
ap.add_argument("--width", type=int, default=1920)
ap.add_argument("--height", type=int, default=1080)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--balance", action="store_true")
ap.add_argument("--radius", type=int, default=7)
ap.add_argument("--image", type=int, default=0, help="guided radius; > 0 selects image mode")
a = ap.parse_args()
dev = torch.device("cuda", 0)
scene = Scene(a.width, a.height, 3000, dev)
frames = torch.stack([scene.hazy_u8(f, 3000 + f, 0.6, (0.85, 0.87, 0.9)) for f in range(a.frames)])
params = DehazeParams(resize_to=None, white_balance=a.balance, patch_radius=a.radius,
                      mode="image" if a.image > 0 else "video", guided_radius=max(a.image, 1))
eng = engine_for(dev)
for _ in range(a.iters):
    out, air = eng.run(frames, params)
torch.cuda.synchronize()
print("ok", out.shape, air[0].tolist())
