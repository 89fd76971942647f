"""Throughput of two independent C3 batches replayed concurrently on two streams
(each a captured GraphedPipeline with its own workspace and output) vs one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import GraphedPipeline
from paper_2512_16609_b200.synthetic import make_frames

dev = torch.device("cuda", 0)
n = int(os.environ.get("N", 300))
frames = make_frames("c3", frames=n, device=dev)
p = DehazeParams(resize_to=None)
g1 = GraphedPipeline(frames, p, streams=1)
g2 = GraphedPipeline(frames, p, streams=1)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def one():
    g1.replay()


def two():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        g1.graph.replay()
    with torch.cuda.stream(s2):
        g2.graph.replay()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1 = timed(one)
t2 = timed(two)
print(f"one batch per step: {t1:.4f} ms/batch; two concurrent: {t2 / 2:.4f} ms/batch ({t2:.4f} per pair)")
print("outputs equal:", torch.equal(g1.out, g2.out))
