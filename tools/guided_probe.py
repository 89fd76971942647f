"""Times the image-mode implementations (DHZ_GUIDED_PATH=strip|fused|twopass) on C5 / C2
batches with CUDA events, and checks they agree with each other (<= 1 LSB)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_16609_b200 import DehazeParams
from paper_2512_16609_b200.engine import FrameEngine
from paper_2512_16609_b200.synthetic import make_frames

dev = torch.device("cuda", 0)
cfgs = {
    "c5": (DehazeParams.for_image(patch_radius=15, guided_radius=60, guided_eps=1e-3),
           lambda n: make_frames("c5", frames=n, device=dev), int(os.environ.get("C5N", "8"))),
    "c2": (DehazeParams.for_image(guided_radius=30, guided_eps=1e-3), lambda n: make_frames("c2", frames=n, device=dev), 1),
    "c5nb": (DehazeParams.for_image(patch_radius=15, guided_radius=60, guided_eps=1e-3, white_balance=False),
             lambda n: make_frames("c5", frames=n, device=dev), int(os.environ.get("C5N", "8"))),
}
for name in sys.argv[1:] or ["c5", "c2"]:
    params, mk, n = cfgs[name]
    frames = mk(n)
    res = {}
    outs = {}
    for path in os.environ.get("PATHS", "strip,fused").split(","):
        os.environ["DHZ_GUIDED_PATH"] = path
        eng = FrameEngine(dev)
        for _ in range(2):
            out, air = eng.run(frames, params)
        torch.cuda.synchronize()
        tot = []
        for it in range(3):
            st = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            out, air = eng.run(frames, params, events=st)
            torch.cuda.synchronize()
            tot.append([st[i].elapsed_time(st[i + 1]) for i in range(4)])
        best = min(tot, key=lambda v: sum(v))
        res[path] = dict(ms_total=round(sum(best), 3), stage_ms=[round(v, 3) for v in best])
        outs[path] = out.clone()
    ref = next(iter(outs))
    for path in list(outs)[1:]:
        d = (outs[ref].to(torch.int16) - outs[path].to(torch.int16)).abs()
        res[f"diff_{path}_vs_{ref}"] = [int(d.max()), int((d > 0).sum())]
    print(json.dumps({"config": name, "frames": n, **res}), flush=True)
