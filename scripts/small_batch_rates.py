"""Small-batch latency (configs 2 and 4a, plus 64 / 1024 blocks) of the
library in FSE_LIB_PATH: device time of one plan run (median)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field, grid_blocks


def dt(plan, fr, td="f32", reps=20):
    out = plan.run(fr, tile_dtype=td); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); plan.run(fr, out, tile_dtype=td); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


img2 = torch.from_numpy(field(512, 512, seed=2).astype(np.float32)).cuda()
tl = grid_blocks(512, 512, 16)
b2 = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
res = {"lib": os.path.basename(os.environ.get("FSE_LIB_PATH") or "base")}
for n in (64, 256):
    p = fse.ConcealPlan(b2[:n], 512, 512, fse.Geometry(16, 16, 64), gamma=0.5, iterations=100)
    res[f"F64_{n}_us"] = dt(p, img2)
img4 = torch.from_numpy(field(512, 512, seed=4).astype(np.float32)).cuda()
t4 = np.array([(16 * i, 16 * j) for i in range(32) for j in range(32)], np.int32)[::2][:500]
b4 = np.concatenate([np.zeros((len(t4), 1), np.int32), t4], 1)
p = fse.ConcealPlan(b4, 512, 512, fse.Geometry(8, 8, 32), gamma=0.5, iterations=100)
res["F32_500_us"] = dt(p, img4)
print(json.dumps(res))
