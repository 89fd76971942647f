"""dehaze_host_batch end-to-end time vs chunk size (frames per H2D/pipeline/D2H step)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.pipeline import dehaze_host_batch
from paper_2512_16609_b200.synthetic import make_frames

dev = torch.device("cuda", 0)
cfgs = {
    "c4": (DehazeParams(resize_to=None, white_balance=True), "c4", 120, [1, 2, 3, 4, 6]),
    "c3": (DehazeParams(resize_to=None), "c3", 300, [4, 7, 10, 16, 32]),
}
for name in sys.argv[1:] or ["c4", "c3"]:
    p, gen, n, chunks = cfgs[name]
    f = make_frames(gen, frames=n, device=dev).cpu().pin_memory()
    H, W = f.shape[1], f.shape[2]
    for ch in chunks:
        for _ in range(2):
            dehaze_host_batch(f, p, chunk=ch)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            dehaze_host_batch(f, p, chunk=ch)
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"{name} chunk={ch:3d} {t*1e3:8.2f} ms  {n*H*W/t/1e6:9.1f} MP/s", flush=True)
