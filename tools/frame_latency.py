"""Per-call latency of dehaze_frame on numpy 1080p frames (the reference's per-frame API)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams, dehaze_frame, dehaze_image
from paper_2512_16609_b200.synthetic import make_frames

frames = [f.numpy() for f in make_frames("c3", frames=40, device="cuda").cpu()]
for name, fn in (("video native", lambda f: dehaze_frame(f, DehazeParams(resize_to=None))),
                 ("video default (resize)", lambda f: dehaze_frame(f)),
                 ("image (guided r=40, balance)", lambda f: dehaze_image(f))):
    for f in frames[:3]:
        fn(f)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for f in frames:
        fn(f)
    el = (time.perf_counter() - t0) / len(frames)
    print(f"dehaze_frame {name}: {el * 1e3:.2f} ms per 1080p frame")
