import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from golden_cases import pipeline_cases
from paper_2512_16609_b200 import DehazeParams, FrameTelemetry, dehaze_frame
C = pipeline_cases()
for name, c in sorted(C.items()):
    p = DehazeParams(**c["params"])
    for i, f in enumerate(c["frames"][:1]):
        tel = FrameTelemetry(capture_maps=True)
        out = dehaze_frame(f, p, tel)
        dd = np.abs(tel.maps["dark"] - c["dark"][i])
        bad = np.argwhere(dd > 0)
        print(name, "dark maxdiff", dd.max(), "nbad", len(bad), bad[:3].tolist(),
              "air", np.abs(tel.airlights[0] - c["airlight"][i]).max(),
              "tc", np.abs(tel.maps["transmission_coarse"] - c["transmission_coarse"][i]).max(),
              "t", np.abs(tel.maps["transmission"] - c["transmission"][i]).max(),
              "out", np.abs(out.astype(int) - c["out"][i].astype(int)).max(), (out != c["out"][i]).sum())
        if len(bad):
            y, x = bad[0]
            print("   got", tel.maps["dark"][y, x] * 255, "want", c["dark"][i][y, x] * 255)
