"""fp64 reference-arithmetic path: config 1 (one window) and config 2 (256
windows) device time of the image-level plan (CUDA events, median), the
per-iteration slope (I = 1 vs 201), and the wall time of one drop-in
extrapolate_cfse call (host arrays in, result with model + trace out)."""
import json, os, statistics, sys, time
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


img = field(256, 256, seed=1)
img1 = torch.from_numpy(img).cuda()
res = {}
for it in (1, 100, 201):
    p1 = fse.ConcealPlan(np.array([[0, 120, 120]], np.int32), 256, 256, fse.Geometry(16, 16, 64),
                         iterations=it, precision="fp64")
    res[f"config1_I{it}_us"] = t(p1, img1)
res["per_iteration_us"] = (res["config1_I201_us"] - res["config1_I1_us"]) / 200
res["config1_us"] = res.pop("config1_I100_us")
img2 = torch.from_numpy(field(512, 512, seed=2)).cuda()
tl = grid_blocks(512, 512, 16)
b2 = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
p2 = fse.ConcealPlan(b2, 512, 512, fse.Geometry(16, 16, 64), iterations=100, precision="fp64")
res["config2_fp64_us"] = t(p2, img2, 5)
res["config2_fp64_blocks_per_s"] = 256 / (res["config2_fp64_us"] * 1e-6)
s = img[96:160, 96:160].copy()
mask = fse.build_mask((64, 64), (24, 24, 16, 16), 16)
cfg = fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=100)
fse.extrapolate_cfse(s, mask, cfg)
ws = []
for _ in range(20):
    t0 = time.perf_counter(); fse.extrapolate_cfse(s, mask, cfg); ws.append(time.perf_counter() - t0)
res["extrapolate_cfse_call_ms"] = statistics.median(ws) * 1e3
print(json.dumps(res))
