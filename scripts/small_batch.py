"""Small-batch latency: config 2 (256 blocks, F=64) and 4b (500 blocks, F=128)
device time per plan run, for variant libraries (FSE_LIB_PATH)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field, grid_blocks


def t(plan, fr, td="f32", reps=30):
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
res = {}
for n in (64, 256):
    p = fse.ConcealPlan(b2[:n], 512, 512, fse.Geometry(16, 16, 64), iterations=100)
    res[f"F64_n{n}_us"] = t(p, img2)
imgs = torch.from_numpy(np.stack([field(512, 512, seed=40 + k) for k in range(8)]).astype(np.float32)).cuda()
b4b = np.array([(f, 64 * i, 64 * j) for f in range(8) for i in range(8) for j in range(8)], np.int32)[:500]
res["F128_n500_us"] = t(fse.ConcealPlan(b4b, 512, 512, fse.Geometry(32, 16, 128), iterations=100), imgs)
print(json.dumps(res))
