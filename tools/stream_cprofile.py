"""cProfile of process_stream (native size, 120 frames of 1080p)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16609_b200 import DehazeParams, process_stream
from paper_2512_16609_b200.synthetic import make_frames

frames = [f.numpy() for f in make_frames("c3", frames=120, device="cuda").cpu()]
p = DehazeParams(resize_to=None)
process_stream(frames[:4], p, sink=lambda o: None)
pr = cProfile.Profile()
pr.enable()
process_stream(frames, p, sink=lambda o: None)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
