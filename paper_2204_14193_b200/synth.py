"""Seeded synthetic inputs standing in for the paper's test images.

The paper evaluates on Kodak / Lena / Baboon / Peppers,
none of which are available here.  BASELINE.json's configs replace them with
seeded 1/f^2 Gaussian random fields (plus straight edges for the video-like
configs 3 and 5); the recipe is SURVEY.md section 8(d):

* field(H, W, seed): amplitude 1/|f| (f from fftfreq, A(0,0) = 0), phase
  U[0, 2pi) from numpy's default_rng(seed), x = Re(ifft2(A e^{i theta})),
  standardised to mean 128 / std 40, clipped to [0, 255].
* add_edges: 8 half-plane steps per frame, point uniform in the frame,
  angle U[0, pi), height U[20, 80]; clip and rint to uint8.
* Loss patterns come from the native planner (`fse_loss_pattern` in the
  C-ABI library): seeded random-sequential selection on the block grid
  rejecting 8-adjacent blocks.

`field_torch` is the on-device variant used by bench.py for the box-scale
configs (256 frames of 3840x2160 would take minutes in numpy); it follows
the same recipe with torch's generator, so its values differ from numpy's
for the same seed but its statistics do not.
"""
from __future__ import annotations

import math

import numpy as np


def field(H: int, W: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.fftfreq(W)[None, :]
    f = np.hypot(fy, fx)
    A = np.zeros_like(f)
    nz = f > 0
    A[nz] = 1.0 / f[nz]
    theta = rng.uniform(0.0, 2.0 * np.pi, (H, W))
    x = np.real(np.fft.ifft2(A * np.exp(1j * theta)))
    x = (x - x.mean()) / x.std() * 40.0 + 128.0
    return np.clip(x, 0.0, 255.0)


def add_edges(x: np.ndarray, seed: int, n_edges: int = 8) -> np.ndarray:
    rng = np.random.default_rng(seed + 0x5EED)
    H, W = x.shape
    yy, xx = np.mgrid[0:H, 0:W]
    out = x.astype(np.float64).copy()
    for _ in range(n_edges):
        x0, y0 = rng.uniform(0, W), rng.uniform(0, H)
        th = rng.uniform(0, np.pi)
        h = rng.uniform(20, 80)
        out[(xx - x0) * np.cos(th) + (yy - y0) * np.sin(th) > 0] += h
    return np.rint(np.clip(out, 0, 255)).astype(np.uint8)


def frame_u8(H: int, W: int, seed: int) -> np.ndarray:
    """1/f^2 field plus 8 edges, uint8 (configs 3 and 5)."""
    return add_edges(field(H, W, seed), seed)


def field_torch(n: int, H: int, W: int, seed: int, device, edges: bool = True, u8: bool = True):
    """On-device batch of n frames (torch), same recipe as field/add_edges.
    Frame i is drawn from its own generator seeded with seed + i, so frame f
    of a job is the same whichever rank (or batch) generates it."""
    import torch

    g = torch.Generator(device=device)
    fy = torch.fft.fftfreq(H, device=device, dtype=torch.float64)[:, None]
    fx = torch.fft.fftfreq(W, device=device, dtype=torch.float64)[None, :]
    f = torch.hypot(fy, fx)
    A = torch.where(f > 0, 1.0 / torch.where(f > 0, f, torch.ones_like(f)), torch.zeros_like(f))
    out = torch.empty((n, H, W), dtype=torch.uint8 if u8 else torch.float32, device=device)
    yy = torch.arange(H, device=device, dtype=torch.float32)[:, None]
    xx = torch.arange(W, device=device, dtype=torch.float32)[None, :]
    for i in range(n):
        g.manual_seed(seed + i)
        theta = torch.rand((H, W), generator=g, device=device, dtype=torch.float64) * (2 * math.pi)
        x = torch.fft.ifft2(A * torch.polar(torch.ones_like(theta), theta)).real
        x = ((x - x.mean()) / x.std() * 40.0 + 128.0).clamp_(0, 255).float()
        if edges:
            p = torch.rand((8, 4), generator=g, device=device, dtype=torch.float64).float()
            for e in range(8):
                x0, y0 = p[e, 0] * W, p[e, 1] * H
                th = p[e, 2] * math.pi
                h = 20 + 60 * p[e, 3]
                x += h * (((xx - x0) * torch.cos(th) + (yy - y0) * torch.sin(th)) > 0).float()
        x = x.clamp_(0, 255)
        out[i] = torch.round(x).to(torch.uint8) if u8 else x
    return out


def grid_blocks(H: int, W: int, B: int, step_i: int = 2, step_j: int = 2, offset: int = 0):
    """Blocks at (step*B*i + offset, step*B*j + offset) -- config 2 uses
    every (2i, 2j) block position of a 512x512 image."""
    out = []
    for i in range(0, (H - offset) // (B * step_i) + 1):
        for j in range(0, (W - offset) // (B * step_j) + 1):
            t, l = offset + i * step_i * B, offset + j * step_j * B
            if t + B <= H and l + B <= W:
                out.append((t, l))
    return np.asarray(out, np.int32).reshape(-1, 2)
