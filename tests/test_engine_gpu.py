"""FrameEngine buffer contracts (the ABI writes through raw device pointers).

* caller-supplied ``out`` / ``airlight`` are checked for shape, dtype, device and
  contiguity before any launch, including the resized working size;
* the default output of StreamedEngine / GraphedPipeline has the working size;
* one engine used from two streams: the second run waits for the first run's
  kernels before it reuses the shared workspace (results stay exact);
* frames on a device other than the current one are processed on their device.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _frames(n=3, w=96, h=64):
    from paper_2512_16609_b200.synthetic import make_frames

    return make_frames("c3", frames=n, width=w, height=h, device="cuda")


def test_out_buffer_validation():
    from paper_2512_16609_b200 import DehazeParams
    from paper_2512_16609_b200.engine import FrameEngine

    eng = FrameEngine(torch.device("cuda", 0))
    f = _frames()
    p = DehazeParams(resize_to=(48, 40))
    bad = [torch.empty_like(f),                                             # native size, not the working size
           torch.empty((3, 40, 48, 3), dtype=torch.int16, device="cuda"),   # dtype
           torch.empty((3, 40, 48, 3), dtype=torch.uint8),                  # host
           torch.empty((3, 48, 40, 3), dtype=torch.uint8, device="cuda")[:, :, :, :]
           .transpose(1, 2)]                                                # non-contiguous
    for o in bad:
        with pytest.raises(ValueError, match="out must be"):
            eng.run(f, p, out=o)
    with pytest.raises(ValueError, match="airlight must be"):
        eng.run(f, p, airlight=torch.empty((3, 3), dtype=torch.float32, device="cuda"))
    out, air = eng.run(f, p, out=torch.empty((3, 40, 48, 3), dtype=torch.uint8, device="cuda"))
    assert out.shape == (3, 40, 48, 3) and air.shape == (3, 3)


def test_default_outputs_have_working_size():
    from paper_2512_16609_b200 import DehazeParams
    from paper_2512_16609_b200.engine import FrameEngine, GraphedPipeline, StreamedEngine

    f = _frames(4)
    p = DehazeParams(resize_to=(40, 32))
    want, air = FrameEngine(f.device).run(f, p)
    out, a2 = StreamedEngine(f.device, streams=2).run(f, p, chunk=2)
    torch.cuda.synchronize()
    assert out.shape == (4, 32, 40, 3) and torch.equal(out, want) and torch.equal(a2, air)
    g = GraphedPipeline(f, p, streams=1)
    out, a3 = g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want) and torch.equal(a3, air)


def test_workspace_reuse_across_streams():
    from paper_2512_16609_b200 import DehazeParams
    from paper_2512_16609_b200.engine import FrameEngine

    p = DehazeParams(resize_to=None)
    big = _frames(24, 640, 360)
    small = _frames(2, 640, 360)[:, :, :, [2, 1, 0]].contiguous()
    eng = FrameEngine(big.device)
    want_big, wa_big = eng.run(big, p)
    want_small, wa_small = eng.run(small, p)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        o1 = torch.empty_like(want_big)
        o2 = torch.empty_like(want_small)
        eng.run(big, p, out=o1, stream=s1)       # long run on s1 ...
        eng.run(small, p, out=o2, stream=s2)     # ... the s2 run must not overwrite its workspace
        torch.cuda.synchronize()
        assert torch.equal(o1, want_big) and torch.equal(o2, want_small)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_frames_on_non_current_device():
    from paper_2512_16609_b200 import DehazeParams, dehaze_batch

    p = DehazeParams(resize_to=None)
    f0 = _frames(2)
    want, air = dehaze_batch(f0, p)
    f1 = f0.to("cuda:1")
    with torch.cuda.device(0):
        out, a1 = dehaze_batch(f1, p)
    assert out.device == f1.device
    assert torch.equal(out.cpu(), want.cpu()) and torch.equal(a1.cpu(), air.cpu())
