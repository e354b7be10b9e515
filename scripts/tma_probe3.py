import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
F, B, border = 32, 8, 8
frames = field_torch(1, 540, 960, seed=9, device="cuda", edges=True)
for bl in ([[0, 0, 56]], [[0, 0, 176]], [[0, 200, 176]], [[0, 200, 176], [0, 200, 400]], [[0, 0, 56], [0, 200, 400]]):
    plan = fse.ConcealPlan(np.array(bl, np.int32), 540, 960, fse.Geometry(B, border, F), iterations=1)
    try:
        plan.run(frames, tile_dtype="f32"); torch.cuda.synchronize(); print("ok", bl, flush=True)
    except Exception as e:
        print("FAIL", bl, str(e)[:80], flush=True); break
