"""F = 128: warp-specialised CTA (default) vs the plain kernel (FSE_WS128=0):
identical traces (same spectrum arithmetic and loop), tiles equal up to the
synthesis summation order, and the rates (large batch on 4K u8 frames and
config 4b)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field, field_torch


def run(ws, frames, blocks, H, W, reps=3):
    os.environ["FSE_WS128"] = ws
    plan = fse.ConcealPlan(blocks, H, W, fse.Geometry(32, 16, 128), gamma=0.5, iterations=100)
    t, tr = plan.run(frames, tile_dtype="f32", trace=True)
    torch.cuda.synchronize()
    ts = []
    out = plan.run(frames)
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); plan.run(frames, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return plan.info, t.cpu().numpy(), tr["uv"].cpu().numpy(), tr["c"].cpu().numpy(), statistics.median(ts)


frames = field_torch(16, 2160, 3840, seed=9, device="cuda", edges=True)
blocks = fse.frames_pattern(16, 2160, 3840, 32, 0.04, seed=2)
imgs = torch.from_numpy(np.stack([field(512, 512, seed=40 + k) for k in range(8)]).astype(np.float32)).cuda()
b4b = np.array([(f, 64 * i, 64 * j) for f in range(8) for i in range(8) for j in range(8)], np.int32)[:500]
res = {}
for name, fr, bl, H, W in (("4k_u8", frames, blocks, 2160, 3840), ("config4b", imgs, b4b, 512, 512)):
    i1, t1, u1, c1, ms1 = run("1", fr, bl, H, W)
    i0, t0, u0, c0, ms0 = run("0", fr, bl, H, W)
    res[name] = {"blocks": len(bl), "ws_threads": i1["threads"], "plain_threads": i0["threads"],
                 "traces_equal": bool(np.array_equal(u1, u0) and np.array_equal(c1, c0)),
                 "max_tile_diff": float(np.abs(t1 - t0).max()), "ws_ms": ms1, "plain_ms": ms0,
                 "ws_blocks_per_s": len(bl) / ms1 * 1e3, "plain_blocks_per_s": len(bl) / ms0 * 1e3,
                 "ws_frac_nominal": len(bl) / ms1 * 1e3 * 8 * 128 * 128 * 100 / (148 * 128 * 1965e6)}
os.environ.pop("FSE_WS128")
print(json.dumps(res))
