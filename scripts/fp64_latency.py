"""fp64 reference-arithmetic path: config 1 (one window) and config 2 (256
windows) device time of the image-level plan (CUDA events, median)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field, grid_blocks


def t(plan, fr, reps=20):
    out = plan.run(fr, tile_dtype="f64"); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); plan.run(fr, out, tile_dtype="f64"); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


img1 = torch.from_numpy(field(256, 256, seed=1)).cuda()
p1 = fse.ConcealPlan(np.array([[0, 120, 120]], np.int32), 256, 256, fse.Geometry(16, 16, 64), iterations=100,
                     precision="fp64")
img2 = torch.from_numpy(field(512, 512, seed=2)).cuda()
tl = grid_blocks(512, 512, 16)
b2 = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
p2 = fse.ConcealPlan(b2, 512, 512, fse.Geometry(16, 16, 64), iterations=100, precision="fp64")
print(json.dumps({"config1_us": t(p1, img1), "config2_fp64_us": t(p2, img2, 5)}))
