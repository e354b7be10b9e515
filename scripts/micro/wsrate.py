import os, sys, json, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
frames = field_torch(16, 2160, 3840, seed=9, device="cuda", edges=True)
blocks = fse.frames_pattern(16, 2160, 3840, 32, 0.04, seed=2)
plan = fse.ConcealPlan(blocks, 2160, 3840, fse.Geometry(32, 16, 128), gamma=0.5, iterations=100)
out = plan.run(frames); torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.run(frames, out); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(os.environ.get("FSE_LIB_PATH", "base")[-12:], os.environ.get("FSE_WS128"), plan.info["threads"], len(blocks) / statistics.median(ts) * 1e3)
