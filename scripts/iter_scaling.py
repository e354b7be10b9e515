"""Per-block fixed cost vs per-iteration cost of the fused kernel: time the
same blocks at several iteration counts (t(I) = C + I L)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
nf, H, W = 64, 2160, 3840
frames = field_torch(nf, H, W, seed=3, device="cuda")
blocks = fse.frames_pattern(nf, H, W, 16, 0.05, 5)
res = []
for I in (25, 50, 100, 200, 400):
    plan = fse.ConcealPlan(blocks, H, W, iterations=I)
    t = plan.run(frames); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): plan.run(frames, t)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    res.append((I, ms))
    print(f"I={I:4d}: {ms:8.3f} ms  {len(blocks) / ms / 1e3:8.3f} Mblk/s  {ms * 1e6 / len(blocks) * 148 * 5 / I:7.3f} ns/iter/slot")
I = np.array([r[0] for r in res], float); T = np.array([r[1] for r in res])
L, C = np.polyfit(I, T, 1)
print(f"fit: per-iteration {L:.4f} ms, fixed {C:.3f} ms -> setup+synthesis = {C / L:.1f} iteration-equivalents")
