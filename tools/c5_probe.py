"""C5-scale image-mode parity probe: GPU output vs the CPU oracle on W >= 4096 frames.

Runs (a) 4096x160 frames, guided r=60, patch 15, balance on and off and (b) one full
BASELINE C5 frame (7680x4320, patch_radius=15, guided_radius=60, eps=1e-3, balance on),
and prints the airlight match, the number of differing output samples and the max
difference.  Test infrastructure (imports the oracle)."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import dehaze_oracle
from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import engine_for
from paper_2512_16609_b200.synthetic import make_frames

dev = torch.device("cuda", 0)
full = "--full" in sys.argv
cases = []
for bal in (True, False):
    cases.append(("4096x160 bal=%d" % bal, DehazeParams.for_image(patch_radius=15, guided_radius=60, guided_eps=1e-3,
                                                                  white_balance=bal),
                  make_frames("c5", frames=2, width=4096, height=160)))
if full:
    cases.append(("c5 full", DehazeParams.for_image(patch_radius=15, guided_radius=60, guided_eps=1e-3),
                  make_frames("c5", frames=1, device=dev).cpu()))
res = []
for name, params, frames in cases:
    t0 = time.time()
    out, air = engine_for(dev).run(frames.to(dev), params)
    torch.cuda.synchronize()
    out = out.cpu().numpy(); air = air.cpu().numpy()
    for i in range(frames.shape[0]):
        maps = {}
        t1 = time.time()
        want = dehaze_oracle.dehaze_frame(frames[i].numpy(), params, maps)
        d = np.abs(out[i].astype(np.int16) - want.astype(np.int16))
        r = dict(case=name, frame=i, airlight_exact=bool(np.array_equal(air[i], maps["airlight"])),
                 max_diff=int(d.max()), n_diff=int((d > 0).sum()), oracle_s=round(time.time() - t1, 1))
        print(json.dumps(r), flush=True)
        res.append(r)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/c5_probe.json", "w") as f:
    json.dump(res, f, indent=1)
