"""Oracle vs the live reference on fresh seeded inputs (only where /root/reference exists)."""
import importlib.util
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src/dehaze"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")


@pytest.fixture(scope="module")
def ref():
    spec = importlib.util.spec_from_file_location("dehaze_ref_t", os.path.join(REF, "__init__.py"),
                                                  submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["dehaze_ref_t"] = mod
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("seed", range(6))
def test_random_frames_all_modes(oracle, ref, seed):
    rng = np.random.default_rng(500 + seed)
    h, w = int(rng.integers(8, 50)), int(rng.integers(8, 60))
    f = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    for p in (ref.DehazeParams(resize_to=None, patch_radius=int(rng.integers(1, 6))),
              ref.DehazeParams(resize_to=(int(rng.integers(4, 40)), int(rng.integers(4, 40)))),
              ref.DehazeParams.for_image(guided_radius=int(rng.integers(1, 6))),
              ref.DehazeParams(resize_to=None, white_balance=True, gamma=1.0)):
        tel = ref.FrameTelemetry(capture_maps=True)
        want = ref.dehaze_frame(f, p, tel)
        maps = {}
        got = oracle.dehaze_frame(f, p, maps)
        assert np.array_equal(got, want)
        assert np.array_equal(maps["airlight"], tel.airlights[0])
