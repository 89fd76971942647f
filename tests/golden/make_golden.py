"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the survey container, where the reference package exists read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference (/root/reference/pkg/src/dehaze) is imported under the alias
``dehaze_ref``; it is not needed afterwards: the committed .npz files pin the
CPU oracle (tests/test_oracle_golden.py, ``-m "not gpu"``) and the CUDA path
(tests/test_golden_gpu.py) on the GPU box, where /root/reference is absent.
All inputs are seeded; sizes are kept small so the fixtures stay < 2 MB.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src/dehaze"


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "dehaze_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["dehaze_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def params_dict(p):
    return {k: getattr(p, k) for k in ("mode", "patch_radius", "top_fraction", "alpha", "omega", "t_min",
                                       "guided_radius", "guided_eps", "gamma", "white_balance", "resize_to")}


def frame_cases(ref):
    """(name, frames (n,H,W,3) u8, params) — pipeline cases."""
    sys.path.insert(0, ROOT)
    from paper_2512_16609_b200.synthetic import make_frames

    rng = np.random.default_rng(2024)
    P = ref.DehazeParams
    syn = make_frames("c3", frames=3, width=128, height=96).numpy()
    syn4k = make_frames("c4", frames=2, width=96, height=64).numpy()
    syn5 = make_frames("c5", frames=1, width=80, height=64).numpy()
    blocks = np.zeros((2, 60, 80, 3), np.uint8)
    for i in range(2):
        r = np.random.default_rng(60 + i)
        clean = np.zeros((60, 80, 3))
        for _ in range(10):
            y, x = int(r.integers(0, 54)), int(r.integers(0, 74))
            bh, bw = int(r.integers(5, 30)), int(r.integers(5, 40))
            clean[y:y + bh, x:x + bw] = r.uniform(0.0, 0.9, size=3)
        hazy = ref.compose_haze(np.clip(clean, 0, 1), ref.HazeSpec(airlight=(0.8, 0.8, 0.8), transmission=0.5))
        blocks[i] = ref.float_to_u8(hazy)
    return [
        ("video_synth", syn, P(resize_to=None)),
        ("video_synth_gamma1", syn[:1], P(resize_to=None, gamma=1.0, omega=1.0, alpha=1.0)),
        ("video_random_odd", rng.integers(0, 256, size=(2, 37, 53, 3), dtype=np.uint8), P(resize_to=None)),
        ("video_random_r3", rng.integers(0, 256, size=(2, 32, 48, 3), dtype=np.uint8),
         P(resize_to=None, patch_radius=3, top_fraction=0.01)),
        ("video_black_white", np.stack([np.zeros((24, 30, 3), np.uint8), np.full((24, 30, 3), 255, np.uint8)]),
         P(resize_to=None)),
        ("video_top_all", rng.integers(0, 256, size=(1, 16, 20, 3), dtype=np.uint8),
         P(resize_to=None, top_fraction=1.0, alpha=1.0)),
        ("video_balance", syn4k, P(resize_to=None, white_balance=True)),
        ("video_resize", syn[:2], P(resize_to=(64, 48))),
        ("video_resize_up", rng.integers(0, 256, size=(1, 20, 26, 3), dtype=np.uint8), P(resize_to=(40, 30))),
        ("image_blocks", blocks, P.for_image(guided_radius=8)),
        ("image_synth_r15", syn5, P.for_image(patch_radius=15, guided_radius=12, guided_eps=1e-3)),
        ("image_nobalance", syn[:1], P.for_image(guided_radius=5, white_balance=False, t_min=0.2)),
    ]


def main():
    ref = load_reference()
    out = {}
    for name, frames, params in frame_cases(ref):
        res = {"frames": frames, "params": np.array(repr(params_dict(params)))}
        outs, airs, darks, tco, tfi = [], [], [], [], []
        for f in frames:
            tel = ref.FrameTelemetry(capture_maps=True)
            outs.append(ref.dehaze_frame(f, params, tel))
            airs.append(tel.airlights[0])
            darks.append(tel.maps["dark"])
            tco.append(tel.maps["transmission_coarse"])
            tfi.append(tel.maps["transmission"])
        res["out"] = np.stack(outs)
        res["airlight"] = np.stack(airs)
        res["dark"] = np.stack(darks)
        res["transmission_coarse"] = np.stack(tco)
        res["transmission"] = np.stack(tfi)
        out[name] = res
    np.savez_compressed(os.path.join(HERE, "pipeline_cases.npz"),
                        **{f"{k}__{kk}": vv for k, v in out.items() for kk, vv in v.items()})

    # public float64 stage functions (reference unit-test style inputs)
    rng = np.random.default_rng(7)
    st = {}
    m = rng.random((19, 23))
    img = rng.random((17, 21, 3))
    for r in (0, 1, 3, 9):
        st[f"min_filter_r{r}"] = ref.min_filter(m, r)
        st[f"box_filter_r{r}"] = ref.box_filter(m, r)
    g = rng.random((19, 23))
    st["guided_r2"] = ref.guided_filter(m, g, 2, 1e-3)
    st["guided_r5"] = ref.guided_filter(m, g, 5, 1e-2)
    st["channel_min"] = ref.channel_min(img)
    st["dark_r2"] = ref.dark_channel(img, 2)
    st["airlight"] = ref.estimate_airlight(img, ref.dark_channel(img, 2), 0.05, 0.8)
    st["transmission"] = ref.estimate_transmission(img, st["airlight"], 0.5, 0.05)
    t = rng.uniform(0.1, 1.0, size=(17, 21))
    st["recover"] = ref.recover_radiance(img, st["airlight"], t)
    st["gamma"] = ref.gamma_correct(img, 1.2)
    st["balance"] = ref.gray_world_balance(img)
    st["gray"] = ref.to_grayscale(img)
    st["resize_down"] = ref.resize_bilinear(img, 9, 7)
    st["resize_up"] = ref.resize_bilinear(img, 30, 25)
    st["u8_to_float"] = ref.u8_to_float(rng.integers(0, 256, size=(5, 6, 3), dtype=np.uint8))
    st["float_to_u8"] = ref.float_to_u8(rng.uniform(-0.2, 1.2, size=(5, 6, 3)))
    np.savez_compressed(os.path.join(HERE, "stage_cases.npz"), m=m, img=img, g=g, t=t, **st)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
