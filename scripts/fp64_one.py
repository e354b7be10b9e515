"""One config-1 fp64 plan run (for ncu captures of extrapolate_kernel<double, 0>)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field
it = int(sys.argv[1]) if len(sys.argv) > 1 else 100
img1 = torch.from_numpy(field(256, 256, seed=1)).cuda()
p1 = fse.ConcealPlan(np.array([[0, 120, 120]], np.int32), 256, 256, fse.Geometry(16, 16, 64),
                     iterations=it, precision="fp64")
for _ in range(2):
    p1.run(img1, tile_dtype="f64")
torch.cuda.synchronize()
