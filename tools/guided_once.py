"""One image-mode batch (C5 geometry, DHZ_GUIDED_PATH from the env) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import FrameEngine
from paper_2512_16609_b200.synthetic import make_frames

dev = torch.device("cuda", 0)
n = int(os.environ.get("C5N", "2"))
bal = os.environ.get("BAL", "0") == "1"
p = DehazeParams.for_image(patch_radius=15, guided_radius=60, guided_eps=1e-3, white_balance=bal)
frames = make_frames("c5", frames=n, device=dev)
eng = FrameEngine(dev)
for _ in range(int(os.environ.get("REPS", "2"))):
    out, air = eng.run(frames, p)
torch.cuda.synchronize()
print("ok", out.shape)
