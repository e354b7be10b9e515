"""Device time of one cFSE plan run (F = SWEEP_F, default 64) vs block count (config-5 frames,
u8, I = 100) for the library in FSE_LIB_PATH: where small batches switch
from latency- to throughput-bound."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch

F = int(os.environ.get("SWEEP_F", "64"))
frames = field_torch(4, 2160, 3840, seed=5, device="cuda", edges=True)
allb = fse.frames_pattern(4, 2160, 3840, F // 4, 0.05, seed=5)
rng = np.random.default_rng(0)
res = {"lib": os.path.basename(os.environ.get("FSE_LIB_PATH") or "base"), "F": F, "variant": os.environ.get("FSE_VARIANT", "auto")}
for n in [int(x) for x in (sys.argv[1:] or [128, 256, 512, 768, 1024, 1536, 2048, 3072, 4096])]:
    b = allb[np.sort(rng.choice(len(allb), n, replace=False))]
    p = fse.ConcealPlan(b, 2160, 3840, fse.Geometry(F // 4, F // 4, F), rho_hat=0.8, gamma=0.5, iterations=100)
    out = p.run(frames); torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.run(frames, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    res[str(n)] = round(statistics.median(ts), 1)
print(json.dumps(res))
