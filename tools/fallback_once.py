import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import engine_for
from paper_2512_16609_b200.synthetic import make_frames
dev = torch.device("cuda", 0)
frames = make_frames("c3", frames=300, device=dev)
eng = engine_for(dev)
p = DehazeParams(resize_to=None, top_fraction=float(os.environ.get("TF", "0.3")))
for _ in range(2):
    eng.run(frames, p)
torch.cuda.synchronize()
print("ok")
