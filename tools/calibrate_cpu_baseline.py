"""Calibrate the CPU baseline: the real reference package (/root/reference, this container
only) against the oracle port bench.py times on the GPU box, on identical seeded frames
(one thread each; the same frames through both; outputs compared)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
import numpy as np
from paper_2512_16609_b200.synthetic import make_frames
from oracle import dehaze_oracle

sys.path.insert(0, "/root/reference/pkg/src")
import dehaze as ref  # the REAL reference (sys.path order: reference first for this import)
assert "/root/reference" in ref.__file__, ref.__file__
from dehaze.pipeline import DehazeParams as RefParams, process_stream as ref_stream

res = {}
for cfg, n, kw in (("c3", 4, dict(resize_to=None)), ("c1", 8, dict(resize_to=None)),
                   ("c4", 1, dict(resize_to=None, white_balance=True)),
                   ("c2", 1, dict(mode="image", resize_to=None, guided_radius=30, guided_eps=1e-3))):
    frames = list(make_frames(cfg, frames=n).numpy())
    rp = RefParams(**kw)
    t0 = time.perf_counter()
    outs_r = []
    ref_stream(frames, rp, sink=outs_r.append, workers=1)
    tr = time.perf_counter() - t0
    t0 = time.perf_counter()
    outs_o, _ = dehaze_oracle.process_stream(frames, dehaze_oracle.OracleParams(**kw), workers=1)
    to = time.perf_counter() - t0
    same = all(np.array_equal(a, b) for a, b in zip(outs_r, outs_o))
    npx = frames[0].shape[0] * frames[0].shape[1]
    res[cfg] = dict(frames=n, reference_ms_per_frame=round(1e3 * tr / n, 1), port_ms_per_frame=round(1e3 * to / n, 1),
                    reference_mps=round(n * npx / tr / 1e6, 3), port_mps=round(n * npx / to / 1e6, 3),
                    port_over_reference=round(tr / to, 3), identical_outputs=same)
    print(cfg, res[cfg], flush=True)
res["host"] = dict(cpu_count=os.cpu_count(), numpy=np.__version__, threads=1,
                   note="survey container (8-core Xeon), not the GPU box")
os.makedirs("profiles", exist_ok=True)
with open("profiles/r02_cpu_baseline_calibration.json", "w") as fh:
    json.dump(res, fh, indent=1)
