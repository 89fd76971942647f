import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2512_16609_b200 import DehazeParams, process_stream, dehaze_batch
from paper_2512_16609_b200.pipeline import dehaze_host_batch
from paper_2512_16609_b200.synthetic import make_frames
p = DehazeParams(resize_to=None)
fr = make_frames("c1", frames=1, device="cuda")
def ps(tag):
    frames = [f.numpy() for f in fr.cpu()]
    ts = []
    for it in range(5):
        t0 = time.perf_counter(); process_stream(frames, p, sink=lambda o: None); ts.append((time.perf_counter()-t0)*1e3)
    print(tag, " ".join(f"{t:.2f}" for t in ts), flush=True)
ps("fresh")
dehaze_batch(fr, p); torch.cuda.synchronize()
ps("after batch")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    dehaze_batch(fr, p); torch.cuda.synchronize()
ps("after profiler")
hin = fr.cpu().pin_memory()
dehaze_host_batch(hin, p); torch.cuda.synchronize()
ps("after host batch")
