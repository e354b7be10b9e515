"""Device time of one config-1 fp64 plan run (I = 1 and 100) with the
library in FSE_LIB_PATH (FSE_GDIAG phase builds: setup cut after phase k)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field
img1 = torch.from_numpy(field(256, 256, seed=1)).cuda()
out = {}
for it in (1, 100):
    p1 = fse.ConcealPlan(np.array([[0, 120, 120]], np.int32), 256, 256, fse.Geometry(16, 16, 64),
                         iterations=it, precision="fp64")
    o = p1.run(img1, tile_dtype="f64"); torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p1.run(img1, o, tile_dtype="f64"); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out[f"I{it}_us"] = statistics.median(ts)
print(os.path.basename(os.environ.get("FSE_LIB_PATH") or "base"), json.dumps(out))
