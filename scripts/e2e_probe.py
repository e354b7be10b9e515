"""Probe the host pipeline: raw pinned H2D bandwidth and Concealer.run time per chunk size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
nf, H, W = 64, 2160, 3840
frames = field_torch(nf, H, W, seed=3, device="cuda")
host = frames.cpu().pin_memory()
dev = torch.empty_like(frames)
for _ in range(2): dev.copy_(host, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5): dev.copy_(host, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
print(f"H2D pinned {host.numel() / dt / 1e9:.1f} GB/s")
blocks = fse.frames_pattern(nf, H, W, 16, 0.05, 5)
plan = fse.ConcealPlan(blocks, H, W)
tiles = plan.run(frames); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): plan.run(frames, tiles)
torch.cuda.synchronize(); dk = (time.perf_counter() - t) / 5
print(f"device-only {len(blocks) / dk / 1e6:.3f} Mblk/s ({dk * 1e3:.1f} ms)")
for ch in (8, 16, 32, 64):
    con = fse.Concealer(blocks, nf, H, W, chunk_frames=ch)
    con.run(host)
    t = time.perf_counter()
    for _ in range(3): con.run(host)
    de = (time.perf_counter() - t) / 3
    print(f"chunk {ch}: e2e {len(blocks) / de / 1e6:.3f} Mblk/s ({de * 1e3:.1f} ms)")
