import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
frames = field_torch(16, 2160, 3840, seed=9, device="cuda")
for F, B, bd, frac in ((128, 32, 16, 0.04), (32, 8, 8, 0.05)):
    blocks = fse.frames_pattern(16, 2160, 3840, B, frac, seed=2)
    res = []
    for I in (50, 100, 200):
        plan = fse.ConcealPlan(blocks, 2160, 3840, fse.Geometry(B, bd, F), iterations=I)
        t = plan.run(frames); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); plan.run(frames, t); plan.run(frames, t); e1.record(); torch.cuda.synchronize()
        res.append((I, e0.elapsed_time(e1) / 2))
    I = np.array([r[0] for r in res], float); T = np.array([r[1] for r in res])
    L, C = np.polyfit(I, T, 1)
    print(f"F={F}: {res}  fixed = {C / L:.1f} iteration-equivalents")
