"""Select cost when the top K spans more than 16 levels below the max (full-histogram fallback)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import engine_for
from paper_2512_16609_b200.synthetic import make_frames

dev = torch.device("cuda", 0)
frames = make_frames("c3", frames=300, device=dev)
eng = engine_for(dev)
for tf in (0.001, 0.05, 0.3):
    p = DehazeParams(resize_to=None, top_fraction=tf)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for _ in range(3):
        eng.run(frames, p, events=evs)
    torch.cuda.synchronize()
    st = [evs[i].elapsed_time(evs[i + 1]) for i in range(4)]
    print(f"top_fraction {tf}: stages ms {[round(x, 4) for x in st]}")
