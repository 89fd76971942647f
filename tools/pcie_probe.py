"""PCIe ceiling for the e2e path: pinned H2D / D2H alone and overlapped, and
dehaze_host_batch at several chunk sizes (c3 workload shape)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.pipeline import dehaze_host_batch

dev = torch.device("cuda", 0)
n, H, W = 300, 1080, 1920
nb = n * H * W * 3
h_in = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(nb, dtype=torch.uint8, device=dev)
d_b = torch.empty(nb, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D alone {nb / t / 1e9:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H alone {nb / t / 1e9:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t = timed(both)
print(f"H2D+D2H overlapped: {nb / t / 1e9:.1f} GB/s each way, {t * 1e3:.1f} ms for {nb / 1e9:.2f} GB each")

frames = h_in.view(n, H, W, 3)
out = h_out.view(n, H, W, 3)
air = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
p = DehazeParams(resize_to=None)
for mb in (8, 16, 24, 48, 96, 192):
    chunk = max(1, (mb << 20) // (3 * H * W))
    t = timed(lambda: dehaze_host_batch(frames, p, out=out, airlight=air, chunk=chunk))
    print(f"dehaze_host_batch chunk {chunk:3d} frames ({mb} MiB): {t * 1e3:.1f} ms/step, {n * H * W / t / 1e6:.0f} MP/s")
