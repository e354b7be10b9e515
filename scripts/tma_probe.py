import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
F, B, border = [int(x) for x in sys.argv[1:4]]
frames = field_torch(2, 540, 960, seed=9, device="cuda", edges=True)
blocks = fse.frames_pattern(2, 540, 960, B, 0.05, seed=2)
plan = fse.ConcealPlan(blocks, 540, 960, fse.Geometry(B, border, F), iterations=100)
t = plan.run(frames, tile_dtype="f32"); torch.cuda.synchronize()
os.environ["FSE_TMA"] = "0"
d = plan.run(frames, tile_dtype="f32"); torch.cuda.synchronize()
print(F, "equal", bool((t == d).all()), float((t - d).abs().max()))
