"""One config-2 plan run (256 blocks of a 512x512 f32 field, fused fp32) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field, grid_blocks
img = torch.from_numpy(field(512, 512, seed=2).astype(np.float32)).cuda()
tl = grid_blocks(512, 512, 16)
b = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
plan = fse.ConcealPlan(b, 512, 512, fse.Geometry(16, 16, 64), gamma=0.5, iterations=100)
for _ in range(2):
    plan.run(img, tile_dtype="f32")
torch.cuda.synchronize()
