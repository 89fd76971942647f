"""Seeded synthetic hazy frames for the BASELINE.json configurations.

No public dataset is used by the reference; the BASELINE configs describe a
generator, restated here in torch so it runs on the GPU for
the 1080p/4K/8K bench batches and on the CPU for small parity inputs:

  clean J  = sum of 32 Gaussian colour blobs (centres uniform, sigma ~ U[10, 80] px,
             colour ~ U[0,1]^3) + U[0, 0.05] noise, clipped to [0, 1]
  depth d  = 0.5 + 4.5*y/(H-1) + 0.5*z, z = low-frequency noise (N(0,1) at 1/8
             resolution, Gaussian-blurred with sigma 5 px there, i.e. ~40 px at full
             resolution, bilinearly upsampled, normalised to unit std); d >= 0
  t        = exp(-beta*d);  I = J*t + A*(1-t), quantised like imageops.float_to_u8
Video clips share blobs and depth across frames; blob centres drift +2 px/frame
in x and per-frame noise is re-drawn.  Seeds: clip seed = 1000*config, frame
seed = 1000*config + frame.
"""

from __future__ import annotations

import math

import torch

CONFIGS = {
    # name: (width, height, frames, airlight, beta(f, n) -> float or None for per-image, extra params)
    "c1": dict(width=640, height=480, frames=1, airlight=(0.85, 0.87, 0.90)),
    "c2": dict(width=1920, height=1080, frames=1, airlight=(0.85, 0.87, 0.90)),
    "c3": dict(width=1920, height=1080, frames=300, airlight=(0.85, 0.87, 0.90)),
    "c4": dict(width=3840, height=2160, frames=120, airlight=(0.80, 0.84, 0.92)),
    "c5": dict(width=7680, height=4320, frames=64, airlight=(0.85, 0.87, 0.90)),
}


def _gauss1d(sigma, device):
    rad = int(math.ceil(3 * sigma))
    x = torch.arange(-rad, rad + 1, device=device, dtype=torch.float32)
    k = torch.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def _blur(img, sigma):
    k = _gauss1d(sigma, img.device)
    r = (k.numel() - 1) // 2
    x = img[None, None]
    x = torch.nn.functional.pad(x, (r, r, 0, 0), mode="reflect")
    x = torch.nn.functional.conv2d(x, k.view(1, 1, 1, -1))
    x = torch.nn.functional.pad(x, (0, 0, r, r), mode="reflect")
    x = torch.nn.functional.conv2d(x, k.view(1, 1, -1, 1))
    return x[0, 0]


class Scene:
    """Static scene (blobs + depth) from which drifting frames are rendered."""

    def __init__(self, width, height, seed, device="cpu"):
        self.w, self.h, self.device = width, height, torch.device(device)
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.cx = torch.rand(32, generator=g) * width
        self.cy = torch.rand(32, generator=g) * height
        self.sig = 10.0 + 70.0 * torch.rand(32, generator=g)
        self.col = torch.rand(32, 3, generator=g)
        hs, ws = max(2, height // 8), max(2, width // 8)
        z = torch.randn(hs, ws, generator=g)
        z = _blur(z, 5.0) if min(hs, ws) > 31 else z
        z = torch.nn.functional.interpolate(z[None, None], size=(height, width), mode="bilinear",
                                            align_corners=False)[0, 0]
        z = (z - z.mean()) / z.std().clamp_min(1e-6)
        y = torch.arange(height, dtype=torch.float32)[:, None].expand(height, width)
        d = 0.5 + 4.5 * y / max(1, height - 1) + 0.5 * z
        self.depth = d.clamp_min(0.0).to(self.device)

    def clean(self, frame_idx, seed):
        dev = self.device
        xs = torch.arange(self.w, device=dev, dtype=torch.float32)
        ys = torch.arange(self.h, device=dev, dtype=torch.float32)
        J = torch.zeros(self.h, self.w, 3, device=dev)
        for b in range(32):
            cx = float(self.cx[b]) + 2.0 * frame_idx
            s = float(self.sig[b])
            gx = torch.exp(-0.5 * ((xs - cx) / s) ** 2)
            gy = torch.exp(-0.5 * ((ys - float(self.cy[b])) / s) ** 2)
            J += (gy[:, None] * gx[None, :])[:, :, None] * self.col[b].to(dev)
        g = torch.Generator(device="cpu").manual_seed(seed)
        noise = torch.rand(self.h, self.w, 3, generator=g).to(dev) * 0.05
        return (J + noise).clamp_(0.0, 1.0)

    def hazy_u8(self, frame_idx, seed, beta, airlight):
        J = self.clean(frame_idx, seed)
        t = torch.exp(-beta * self.depth)[:, :, None]
        A = torch.tensor(airlight, device=self.device, dtype=torch.float32)
        I = J * t + A * (1.0 - t)
        return torch.floor(I.clamp(0.0, 1.0) * 255.0 + 0.5).to(torch.uint8)


def make_frames(config="c3", frames=None, width=None, height=None, device="cpu", out=None):
    """Frames of a BASELINE config as a (n, H, W, 3) uint8 tensor on ``device``.

    ``frames``/``width``/``height`` override the config sizes (parity tests use
    small versions of the same generator).
    """
    spec = CONFIGS[config]
    W = width or spec["width"]
    H = height or spec["height"]
    n = frames if frames is not None else spec["frames"]
    ci = int(config[1:])
    if out is None:
        out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=device)
    if config == "c5":
        for f in range(n):
            scene = Scene(W, H, 1000 * ci + f, device)
            g = torch.Generator(device="cpu").manual_seed(1000 * ci + f)
            beta = 0.4 + 0.6 * float(torch.rand(1, generator=g))
            out[f] = scene.hazy_u8(0, 1000 * ci + f, beta, spec["airlight"])
        return out
    scene = Scene(W, H, 1000 * ci, device)
    for f in range(n):
        if config in ("c3", "c4"):
            beta = 0.65 - 0.15 * math.cos(2 * math.pi * f / 300.0)
        else:
            beta = 0.6
        out[f] = scene.hazy_u8(f, 1000 * ci + f, beta, spec["airlight"])
    return out
