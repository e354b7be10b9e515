import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
F, B, border, I, nb = [int(x) for x in sys.argv[1:6]]
frames = field_torch(1, 540, 960, seed=9, device="cuda", edges=True)
blocks = fse.frames_pattern(1, 540, 960, B, 0.05, seed=2)[:nb]
plan = fse.ConcealPlan(blocks, 540, 960, fse.Geometry(B, border, F), iterations=I)
print(plan.info, flush=True)
t = plan.run(frames, tile_dtype="f32"); torch.cuda.synchronize()
print("ok", F, I, nb, flush=True)
