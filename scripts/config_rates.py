"""Per-config measurements (BASELINE.json configs 1-5, SURVEY 8(d) inputs):
device time of one plan run (CUDA events, median of repeats, inputs resident),
lost blocks/s, shared-memory roofline fraction (8 F^2 I bytes per block, SMEM
peak 148 SMs x 128 B/clk x 1965 MHz), and for config 1 the latency of the
drop-in per-window call (host numpy in, ExtrapolationResult out).
Usage: python scripts/config_rates.py > profiles/r01/config_rates.jsonl"""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field, field_torch, grid_blocks

dev = torch.device("cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
PEAK = sms * 128 * 1965e6


def dev_time(fn, reps=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(ts)


def report(name, plan, frames, n, F, I, tile_dtype=None, reps=20, **extra):
    td = tile_dtype or "u8"
    out = plan.run(frames, tile_dtype=td)
    s = dev_time(lambda: plan.run(frames, out, tile_dtype=td), reps)
    rate = n / s
    d = {"config": name, "blocks": n, "F": F, "iterations": I, "device_s": s, "blocks_per_s": rate,
         "smem_frac_nominal": rate * 8 * F * F * I / PEAK, "plan": plan.info}
    if I != 100:
        d["blocks_per_s_100it_equiv"] = rate * I / 100
    if I != 100 or F != 64:  # configs with I != 100 or B != 16
        d["bin_iterations_per_s"] = rate * F * F * I
    d.update(extra)
    print(json.dumps(d), flush=True)


# config 1: one fp64 block at (120, 120) of a 256x256 field
img1 = field(256, 256, seed=1)
b1 = np.array([[0, 120, 120]], np.int32)
p64 = fse.ConcealPlan(b1, 256, 256, fse.Geometry(16, 16, 64), rho_hat=0.8, gamma=0.5, iterations=100,
                      precision="fp64")
fr1 = torch.from_numpy(img1).to(dev)
s = dev_time(lambda: p64.run(fr1, tile_dtype="f64"))
mask = fse.build_mask((64, 64), (24, 24, 16, 16), 16)
win = img1[96:160, 96:160].copy()
cfg = fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=100)
fse.extrapolate_cfse(win, mask, cfg)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); fse.extrapolate_cfse(win, mask, cfg); ts.append(time.perf_counter() - t0)
print(json.dumps({"config": "1 (fp64, one block)", "blocks": 1, "F": 64, "iterations": 100,
                  "plan_device_s": s, "per_window_api_wall_s": statistics.median(ts),
                  "note": "latency-bound: one CTA; the per-window call includes host<->device copies, "
                          "trace and model readback"}), flush=True)

# config 2: 512x512 f32, 256 blocks at (32i, 32j)
img2 = torch.from_numpy(field(512, 512, seed=2).astype(np.float32)).to(dev)
tl = grid_blocks(512, 512, 16)
b2 = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
report("2 (fp32, 256 blocks)", fse.ConcealPlan(b2, 512, 512, fse.Geometry(16, 16, 64), iterations=100, gamma=0.5),
       img2, len(b2), 64, 100, tile_dtype="f32")
p2d = fse.ConcealPlan(b2, 512, 512, fse.Geometry(16, 16, 64), iterations=100, precision="fp64", gamma=0.5)
report("2 (fp64 reference-arithmetic plan, 256 blocks)", p2d, img2.double(), len(b2), 64, 100,
       tile_dtype="f64", reps=5)

# config 3: 64 x 1920x1080 u8 + edges, 10% isolated loss, I = 200
fr3 = field_torch(64, 1080, 1920, seed=3, device=dev, edges=True)
b3 = fse.frames_pattern(64, 1080, 1920, 16, 0.10, seed=3)
report("3 (u8, 64 x 1080p, 10% loss, I=200)",
       fse.ConcealPlan(b3, 1080, 1920, fse.Geometry(16, 16, 64), iterations=200, gamma=0.5), fr3, len(b3), 64, 200,
       reps=5)
del fr3

# config 4a: 500 8x8 blocks, F = 32; 4b: 500 32x32 blocks over 8 images, F = 128
img4 = torch.from_numpy(field(512, 512, seed=4).astype(np.float32)).to(dev)
tl = np.array([(16 * i, 16 * j) for i in range(32) for j in range(32)], np.int32)[::2][:500]
b4a = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
report("4a (fp32, 500 x 8x8, F=32)", fse.ConcealPlan(b4a, 512, 512, fse.Geometry(8, 8, 32), iterations=100, gamma=0.5),
       img4, len(b4a), 32, 100, tile_dtype="f32")
imgs = torch.from_numpy(np.stack([field(512, 512, seed=40 + k) for k in range(8)]).astype(np.float32)).to(dev)
b4b = np.array([(f, 64 * i, 64 * j) for f in range(8) for i in range(8) for j in range(8)], np.int32)[:500]
report("4b (fp32, 500 x 32x32, F=128)",
       fse.ConcealPlan(b4b, 512, 512, fse.Geometry(32, 16, 128), iterations=100, gamma=0.5), imgs, len(b4b), 128, 100,
       tile_dtype="f32")

# config 5: 256 x 4K u8 + edges, 5% loss (the bench workload)
fr5 = field_torch(256, 2160, 3840, seed=5, device=dev, edges=True)
b5 = fse.frames_pattern(256, 2160, 3840, 16, 0.05, seed=5)
report("5 (u8, 256 x 4K, 5% loss)", fse.ConcealPlan(b5, 2160, 3840, fse.Geometry(16, 16, 64), iterations=100, gamma=0.5),
       fr5, len(b5), 64, 100, reps=5)
