"""Small batches through every native path, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck): video at native size (C3-like,
plus a C4-like batch with gray-world balance), image mode (strip kernels and the
one-pass fused kernel, balance on/off), the default resize path and the float64
stage API.  Exits non-zero if any output is inconsistent."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_16609_b200 as dz
from paper_2512_16609_b200 import DehazeParams, dehaze_batch
from paper_2512_16609_b200.synthetic import make_frames

dev = torch.device("cuda", 0)
cases = [
    ("video", DehazeParams(resize_to=None), make_frames("c3", frames=3, width=480, height=272)),
    ("video+balance", DehazeParams(resize_to=None, white_balance=True), make_frames("c4", frames=2, width=384, height=208)),
    ("video odd", DehazeParams(resize_to=None, patch_radius=3), make_frames("c3", frames=2, width=101, height=37)),
    ("image", DehazeParams.for_image(guided_radius=12), make_frames("c2", frames=2, width=256, height=144)),
    ("image wide", DehazeParams.for_image(patch_radius=15, guided_radius=60, white_balance=False),
     make_frames("c5", frames=1, width=4096, height=130)),
    ("resize", DehazeParams(resize_to=(160, 96)), make_frames("c3", frames=2, width=320, height=192)),
    ("resize+balance", DehazeParams(resize_to=(96, 64), white_balance=True), make_frames("c3", frames=2, width=200, height=120)),
]
for path in ("strip", "fused"):
    os.environ["DHZ_GUIDED_PATH"] = path
    for name, p, f in cases:
        if path == "fused" and p.mode != "image":
            continue
        out, air = dehaze_batch(f.to(dev), p)
        torch.cuda.synchronize()
        assert torch.isfinite(air).all(), name
        print(f"{path:5s} {name}: ok", flush=True)
# float64 stage API (floatpath kernels)
rng = np.random.default_rng(1)
img = rng.random((40, 56, 3))
cm = dz.channel_min(img)
dk = dz.min_filter(cm, 3)
A = dz.estimate_airlight(img, dk, 0.01, 0.8)
t = dz.transmission_from_channel_min(cm, A, 0.5, 0.05)
q = dz.guided_filter(t, dz.to_grayscale(img), 5, 1e-3)
r = dz.recover_radiance(img, A, np.maximum(q, 0.05))
g = dz.gray_world_balance(dz.gamma_correct(r, 1.2))
print("float64 stage API: ok", dz.float_to_u8(g).shape)
